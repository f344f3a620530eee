"""Full-size C2 goldens (BASELINE configs[1]: the Fig. 1 reduction on 2^24
ints, 65536 blocks x 256 threads, clean and racy), derived from reference
runs at small sizes -- the reference itself is quadratic in threads and
cannot run 2^24.  Run here:  python tests/make_c2_golden.py

Derivation (each step is checked on the reference runs it uses):
* blocks are independent under round robin and their work does not depend
  on the data (no data-dependent branch), so every per-run count is affine
  in the block count: steps(nb) = a + b * nb, checked on 4 sizes;
* the input in[i] = (21 i + 29) % 100 repeats every 100 ints, so block b's
  partial sum out[b] depends only on b mod 25; the host adds the partials,
  hence OUTPUT(65536 blocks) = 2621 * S(25 blocks) + S(11 blocks) (65536 =
  2621 * 25 + 11), with S(k) the reference OUTPUT at k blocks;
* RaceState::reported of the racy run holds the same (byte, line) pattern in
  every block's shared object, the objects being consecutive from a fixed
  first id -- checked on every block of the sampled runs."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_programs as gp  # noqa: E402
import oracle_bind as ob  # noqa: E402

FULL_BLOCKS = 65536
THREADS = 256


def ref(nb, racy):
    return ob.ref_run(gp.scaled(nb * THREADS, THREADS, racy=racy), "c2.cu", step_limit=10**12, capture=False)


def derive(racy):
    runs = {nb: ref(nb, racy) for nb in (2, 5, 11, 25)}
    xs = sorted(runs)
    b = (runs[xs[1]]["steps"] - runs[xs[0]]["steps"]) // (xs[1] - xs[0])
    a = runs[xs[0]]["steps"] - b * xs[0]
    for nb in xs:
        assert runs[nb]["steps"] == a + b * nb, ("steps not affine in blocks", nb)
        assert runs[nb]["exit"] == (1 if racy else 0)
    s = {nb: int(runs[nb]["output"].split()[-1]) for nb in (11, 25)}
    q, r = divmod(FULL_BLOCKS, 25)
    assert r == 11
    out = {"output": f"OUTPUT: {q * s[25] + s[11]}\n", "steps": a + b * FULL_BLOCKS,
           "exit": runs[25]["exit"], "diags": runs[25]["diags"], "steps_affine": [a, b]}
    if racy:
        pat, first = None, None
        for nb, r_ in runs.items():
            rep = r_["reported"]
            objs = sorted({t[0] for t in rep})
            assert objs == list(range(objs[0], objs[0] + nb)), "consecutive shared objects"
            first = objs[0] if first is None else first
            assert objs[0] == first
            for o in objs:
                p = [[t[1], t[2]] for t in rep if t[0] == o]
                pat = p if pat is None else pat
                assert p == pat, "same pattern in every block"
        out.update({"block_pattern": pat, "first_object": first, "reported": len(pat) * FULL_BLOCKS})
    else:
        assert out["output"] == "OUTPUT: 830472184\n"  # the closed-form sum
    return out


def main():
    gold = {"blocks": FULL_BLOCKS, "threads": THREADS, "clean": derive(False), "racy": derive(True)}
    path = os.path.join(HERE, "golden", "c2_full.json")
    with open(path, "w") as f:
        json.dump(gold, f, separators=(",", ":"), sort_keys=True)
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "block_pattern"} if isinstance(v, dict) else v
                      for k, v in gold.items()}))


if __name__ == "__main__":
    main()
