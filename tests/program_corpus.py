"""The whole-program parity corpus (test infrastructure).

Each entry is (name, filename, source).  The golden RunResults were produced
by the unmodified reference (oracle/_ref/libmckref.so, Machine::run under
--schedule roundrobin) with tests/make_golden.py and are committed in
tests/golden/programs.json, so the GPU box needs no reference build."""
import gen_programs as gp


def corpus():
    out = [
        ("fig1", "sum.cu", gp.fig1()),
        ("fig1_race", "sum_race.cu", gp.fig1_race()),
        ("fig1_deadlock", "dl.cu", gp.fig1_deadlock()),
        ("scaled_256x64", "s.cu", gp.scaled(256 * 4, 256)),
        ("scaled_racy_256x2", "r.cu", gp.scaled(512, 256, racy=True)),
        ("scaled_33x3", "s3.cu", gp.scaled(99, 33)),
        ("scaled_racy_9x4", "r4.cu", gp.scaled(36, 9, racy=True)),
        ("divbar_4x8", "dl4.cu", gp.divergent_barrier_gen(4, 8, 0)),
        ("divbar_6x33", "dl6.cu", gp.divergent_barrier_gen(6, 33, 1)),
        ("divbar_3x64", "dl3.cu", gp.divergent_barrier_gen(3, 64, 2)),
    ]
    for i in range(300):
        out.append((f"rand{i}", f"rand{i}.cu", gp.random_kernel(i)))
    return out


KEYS = ("exit", "output", "steps", "diags", "stuck_reports", "report_text", "reported", "main_return")


def project(run):
    """The fields compared for parity (RunResult + RaceState::reported)."""
    return {k: run.get(k) for k in KEYS}
