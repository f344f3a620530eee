#!/usr/bin/env python3
"""Benchmark of the checker's hot path on B200 (contract: see DESIGN.md §Measurement).

Headline workload (`value`): BASELINE.json configs[2], C3 -- a synthetic
shared-memory access trace of 2^30 events in 2^20 simulated blocks (256
threads x 2 epochs x 2 accesses, 1% injected races), generated on the device.
One step = race detection over the whole trace (mckg_race_out_reset +
mckg_detect_shared, K2); for N > 1 each rank checks its contiguous shard of
blocks and the per-line first-detection table is MIN-all-reduced so rank 0
holds the report order.  This is the HBM-bound race-checked-events path the
north star's roofline target is stated on.

Second workload (`k1` object in the same line): BASELINE.json configs[1], C2
-- the Fig. 1 reduction scaled to 2^24 ints (65536 blocks x 256 threads),
checked end to end through mck_run (result records) (host interpreter + K1 grid engine +
fused race detector): simulated thread-steps/s and race-checked shared
events/s of the grid kernel (CUDA events), plus the whole-program wall time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "race-checked access events/sec and simulated thread-steps/sec, 1/2/4/8 B200 vs CPU"
UNIT = "events/s"
WORKLOAD = ("C3: synthetic shared-memory access trace, 2^30 events, 2^20 blocks x 256 threads, "
            "2 barrier epochs, 1% injected write-write/read-write races")
EVENTS_PER_BLOCK = 1024
FULL_BLOCKS = 1 << 20
BYTES_PER_EVENT = 16
BYTES_PER_BLOCK = 8
BYTES_PER_TRIPLE = 12


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            p = [x.strip() for x in l.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for name, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_replay(n_events_target, nthreads, prefer_ref=True):
    """Time the reference CPU checker (oracle/_ref when present, else the C
    port) on a bounded C3 sample.  Returns (events/s, kind, sample, threads)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob
    nb = max(nthreads, n_events_target // EVENTS_PER_BLOCK)
    ev, bs = ob.gen_c3(0, nb)
    tr = ob.make_trace(ev, bs, ob.C3_SHMEM)
    use_ref = prefer_ref and ob.ref() is not None
    fn = ob.ref_detect if use_ref else ob.port_detect
    t0 = time.perf_counter()
    rc, tri, n, lf = fn(tr, nthreads=nthreads)
    dt = time.perf_counter() - t0
    assert rc == 0
    kind = "reference" if use_ref else "port"
    sample = (f"C3 blocks 0..{nb - 1} ({nb * EVENTS_PER_BLOCK} events, "
              f"{'reference Machine::recordAccess/clearEpoch replay' if use_ref else 'oracle/detector.c'}"
              f", block-partitioned over {nthreads} threads)")
    return nb * EVENTS_PER_BLOCK / dt, kind, sample, nthreads, dt


def calibrate_cpu(nthreads, seconds):
    """Events that take about `seconds` on nthreads host threads."""
    rate1, *_ = cpu_replay(1 << 16, 1)
    return int(min(1 << 28, max(1 << 16, rate1 * nthreads * seconds)))


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    nthreads = host_cores()
    target = calibrate_cpu(nthreads, 3.0)
    for _ in range(args.warmup):
        cpu_replay(target, nthreads)
    vals, times = [], []
    for _ in range(args.steps):
        v, kind, sample, thr, dt = cpu_replay(target, nthreads)
        vals.append(v)
        times.append(dt)
    total_events = (target // EVENTS_PER_BLOCK) * EVENTS_PER_BLOCK * args.steps
    value = total_events / sum(times)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": {"workload": WORKLOAD, "parallelism": f"cpu{thr}",
                                        "sample_events_per_step": total_events // args.steps},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def load_traffic(key="detect_call"):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key)
    except (OSError, ValueError):
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1211_6193_b200 import _abi, race

    ws, rank, local = dist_env()
    # MCKG_BENCH_SHARED_GPU=1: every rank on cuda:0 over gloo -- a functional
    # dry run of the multi-rank paths on a one-GPU box (not a performance mode)
    shared = os.environ.get("MCKG_BENCH_SHARED_GPU") == "1"
    local = 0 if shared else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    blocks = args.blocks
    b0 = blocks * rank // ws
    b1 = blocks * (rank + 1) // ws
    nb = b1 - b0
    ev, bs = race.gen_c3(b0, nb, device=dev)
    tr = race.make_trace(ev, bs, _abi.C3_SHMEM, obj_base=1 + b0, bid_base=b0,
                         max_block_events=EVENTS_PER_BLOCK)
    out = race.RaceOut(capacity=nb * EVENTS_PER_BLOCK // 8, device=dev)
    stream = torch.cuda.current_stream()
    # real multi-GPU: the library's own NCCL communicator does the exchange
    # (mckg_detect_shared_mgpu); the shared-GPU gloo dry run reduces in Python
    comm = None
    if ws > 1 and not shared:
        from paper_1211_6193_b200 import checker
        obj = [checker.comm_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = race.Comm(obj[0], rank, ws, local)
    torch.cuda.synchronize()

    def step(ev0=None, ev1=None):
        out.reset(stream)
        if ev0 is not None:
            ev0.record(stream)
        if comm is not None:
            race.detect_shared_mgpu(comm, tr, out, stream, reset=False)
        else:
            race.detect_shared_async(tr, out, stream, reset=False)
        if ev1 is not None:
            ev1.record(stream)
        if ws > 1 and comm is None:
            lf = out.line_first
            lf.bitwise_xor_(-(1 << 63))  # unsigned order -> signed order
            _all_reduce(lf, dist.ReduceOp.MIN)
            lf.bitwise_xor_(-(1 << 63))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            step(*kevs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    k_ms = [a.elapsed_time(b) for a, b in kevs]
    n_tri = int(out.n_triples.item())
    status = int(out.status.item())
    assert status == 0, f"detector status {status}"
    # the run's own result, sorted into RaceState::reported order on the
    # device, kept on the host for the full-size parity check (cpu leg)
    gpu_res = None
    if (rank == 0 and ws == 1 and not args.no_cpu) or args.dump:
        gpu_res = race.fetch(out, obj_base=1 + b0)
    if args.dump:  # this rank's reported set + the reduced line table (multi-rank set tests)
        import numpy as np
        os.makedirs(args.dump, exist_ok=True)
        np.savez(os.path.join(args.dump, f"c3_r{rank}.npz"), triples=gpu_res.triples,
                 line_first=gpu_res.line_first, n=gpu_res.n_triples)
    if not (rank == 0 and ws == 1 and not args.no_cpu):
        gpu_res = None
    # max over ranks
    t = torch.tensor([ms, statistics.mean(k_ms)], dtype=torch.float64, device=dev)
    tot = torch.tensor([nb * EVENTS_PER_BLOCK, n_tri], dtype=torch.int64, device=dev)
    if ws > 1:
        _all_reduce(t, dist.ReduceOp.MAX)
        _all_reduce(tot, dist.ReduceOp.SUM)
    ms, k_avg = float(t[0]), float(t[1])
    total_events = int(tot[0])
    total_tri = int(tot[1])
    value = total_events * args.steps / (ms / 1e3)
    per_rank_bytes = (nb * EVENTS_PER_BLOCK * BYTES_PER_EVENT + (nb + 1) * BYTES_PER_BLOCK
                      + n_tri * BYTES_PER_TRIPLE)
    achieved = per_rank_bytes / (k_avg / 1e3) / 1e9
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        peak = json.load(open(peaks_path))["hbm_gbs"]
        peak_src = "measured"
    except (OSError, ValueError, KeyError):
        peak, peak_src = 6650.0, "fallback"
    # per step: mckg_race_out_reset (1) + the kernels of the last detect call
    launches = args.steps * (1 + _abi.launch_stats().kernels)

    k1 = None
    if not args.no_k1:
        try:
            k1 = run_k1(args, ws, rank, local, shared)
        except Exception as e:  # noqa: BLE001 -- the C3 line must still print
            k1 = {"error": f"{type(e).__name__}: {e}"[:500]}
    c5 = None
    if not args.no_c5:
        ev = bs = tr = out = None  # free the C3 trace before C5
        torch.cuda.empty_cache()
        # configs[4]: 2^32 events over 8 GPUs = 2^29 per GPU (2^17 blocks of 4096)
        c5 = run_c5(args, args.c5_blocks if args.c5_blocks else (1 << 17) * ws, dev, ws, rank, comm)
    e2e = None
    if rank == 0 and ws == 1 and args.e2e_blocks > 0:
        e2e = run_e2e(args, torch, race, _abi)
    cpu = parity = None
    if gpu_res is not None:
        # the reference CPU checker replays the SAME trace (all of it unless
        # --cpu-blocks bounds it) on every host core: its rate is the CPU
        # baseline, and each chunk is compared with this run's GPU result
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import c3_parity
        nthreads = host_cores()
        cb = args.cpu_blocks if args.cpu_blocks else blocks
        parity = c3_parity.replay_full(gpu_res.triples, gpu_res.line_first, blocks, nthreads, max_blocks=cb)
        parity["gpu_triples"] = int(gpu_res.n_triples)
        cpu = {"value": parity["events"] / parity["replay_s"], "unit": UNIT, "cores": nthreads,
               "cpu_model": cpu_model(), "kind": parity["kind"],
               "sample": (f"C3 blocks 0..{parity['checked_blocks'] - 1} of {blocks} "
                          f"({parity['events']} events; "
                          f"{'reference Machine::recordAccess/clearEpoch' if parity['kind'] == 'reference' else 'oracle/detector.c'}"
                          f" replay, chunks of 2^16 blocks partitioned over {nthreads} threads; "
                          f"generation excluded)")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "events": total_events, "blocks": blocks,
                       "reported_triples": total_tri, "parallelism": f"block-shard{ws}",
                       "parity_checked": bool(parity and parity["checked_blocks"] == parity["of_blocks"]
                                              and parity["triples_equal"] and parity["line_first_equal"]),
                       "l2": "inputs (16 GiB) >> L2 (126 MB); no flush needed"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic(),
                         "kernel": "mckg_detect_shared: fast_kernel (warp per block) + the gated general kernel over its overflow list, timed together", "kernel_ms": k_avg,
                         "peak_source": peak_src,
                         "algorithmic_bytes": "16 B/event + 8 B/block + 12 B/reported triple"},
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
            "k1": k1,
            "c5": c5,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()


def _all_reduce(t, op):
    """all_reduce that also works for CUDA tensors on the gloo dry-run backend."""
    import torch.distributed as dist
    if dist.get_backend() == "gloo" and t.is_cuda:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def run_c5(args, blocks, dev, ws, rank, comm=None):
    """C5 (configs[4]): cross-block global races over `blocks` simulated blocks
    sharded over the ranks: K3 partition -> NCCL all-to-all -> K6 detect ->
    MIN-all-reduce of the line table.  Device-timed (CUDA events), max over
    ranks.  Returns the c5 object of the JSON line (rank 0)."""
    import torch
    import torch.distributed as dist
    from paper_1211_6193_b200 import global_race as gr
    space = blocks * 65536
    b0, b1 = gr.shard(blocks, rank, ws)
    ev = gr.gen_c5(b0, b1 - b0, blocks, device=dev)
    lo, _ = gr.addr_range(rank, ws, space)
    stream = torch.cuda.current_stream()

    outs = {}  # result buffers, allocated once and reused like a caller would

    def out_for(cap):
        if cap not in outs:
            outs[cap] = gr.GlobalOut(cap, device=dev)
        return outs[cap]

    def step():
        if comm is not None:  # the exchange inside the library (mckg_detect_global_mgpu)
            out = out_for(max(1, 2 * ev.shape[0] // 8))
            gr.detect_mgpu(comm, ev, space, out.reset(), stream)
            return out, -1
        if ws > 1:
            grouped, counts = gr.partition(ev, ws, space, stream)
            mine = gr.exchange(grouped, counts)
        else:
            mine = ev  # one owner: nothing to partition or exchange
        out = out_for(max(1, 2 * ev.shape[0] // 8) if ws > 1 else max(1, mine.shape[0] // 8))
        gr.detect(mine, lo, out.reset(), stream)
        if ws > 1:
            out.line_first.bitwise_xor_(-(1 << 63))
            _all_reduce(out.line_first, dist.ReduceOp.MIN)
            out.line_first.bitwise_xor_(-(1 << 63))
        return out, mine.shape[0]

    for _ in range(max(3, args.warmup)):  # the first calls size the stream-ordered pool
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 5))
    t0.record(stream)
    for _ in range(steps):
        out, recv = step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if args.dump:
        import numpy as np
        races, n_r, lf, _ = gr.fetch(out)
        np.savez(os.path.join(args.dump, f"c5_r{rank}.npz"), races=races, line_first=lf, n=n_r)
    n_races = int(out.n.item())
    status = int(out.status.item())
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([ev.shape[0], n_races, max(recv, 0)], dtype=torch.int64, device=dev)
    if ws > 1:
        _all_reduce(t, dist.ReduceOp.MAX)
        _all_reduce(tot, dist.ReduceOp.SUM)
    ms = float(t[0])
    events = int(tot[0])
    sent = ev.shape[0] * 16 * (ws - 1) / max(1, ws)  # bytes leaving this rank (uniform partition)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        peak = json.load(open(peaks_path))["hbm_gbs"]
    except (OSError, ValueError, KeyError):
        peak = 6650.0
    per_rank = ev.shape[0] * 16  # algorithmic: one 16-byte read per record on its rank
    achieved = per_rank / (ms / 1e3) / 1e9
    return {"workload": f"C5: {events} global 4-byte accesses, {blocks} blocks, 1% cross-block, "
                        f"address-range all-to-all over {ws} GPU(s)",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": load_traffic("c5_call") if ws == 1 else None,
                         "kernel": "mckg_detect_global: tile path (span sample, tile_claim, tile_detect, "
                         "tile_multi; side list through the bucket pipeline)"
                         + (" + K3 partition + NCCL all-to-all" if ws > 1 else ""),
                         "algorithmic_bytes": "16 B/event read (+ (P-1)/P x 16 B/event over NVLink at P ranks)"},
            "events_per_s": events / (ms / 1e3), "ms_per_step": ms, "races_reported": int(tot[1]),
            "status": status, "nvlink_bytes_per_rank": sent,
            "nvlink_GBps_per_rank": sent / (ms / 1e3) / 1e9 if ws > 1 else None,
            "parity": "unpinned (no reference semantics); checker oracle/global_detector.c"}


def _k1_run(src, name, ws, rank, dev, shared):
    """One whole-checker run; with ws > 1 every rank runs its block range of
    each grid (NCCL transport; host transport in the shared-GPU dry run)."""
    from paper_1211_6193_b200 import checker
    kw = {}
    if ws > 1:
        import torch.distributed as dist
        kw = dict(rank=rank, world=ws, device=dev)
        if shared:
            kw["allgather"] = checker.torch_allgather()
        else:
            obj = [checker.comm_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            kw["comm"] = obj[0]
    t0 = time.perf_counter()
    # the result-record ABI (no JSON): the end-to-end time is the checker's
    r = checker.run(src, name, step_limit=8_000_000_000, stuck_lists=64, **kw)
    return r, time.perf_counter() - t0


def run_k1(args, ws=1, rank=0, dev=0, shared=False):
    """C2 (configs[1]) and C4 (configs[3]) through the whole checker: K1
    thread-steps/s (device steps / max-over-ranks grid time)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import gen_programs as gp
    src = gp.scaled(1 << 24, 256, racy=args.k1_racy)
    r, wall = _k1_run(src, "c2.cu", ws, rank, dev, shared)
    st = r["stats"]
    gs = max(st["grid_ms"], 1e-6) / 1e3
    ok = (r["output"] == "OUTPUT: 830472184\n" and r["exit"] == 0) if not args.k1_racy else r["exit"] == 1
    out = {"workload": "C2: Fig. 1 reduction, 2^24 ints, 65536 blocks x 256 threads"
                       + (" (racy variant)" if args.k1_racy else ""),
           "parallelism": f"block-range shard over {ws} rank(s)",
           "thread_steps_per_s": st["device_steps"] / gs, "shared_events_per_s": st["shared_events"] / gs,
           "grid_ms": st["grid_ms"], "device_steps": st["device_steps"], "barrier_rules": st["barrier_rules"],
           "shared_events": st["shared_events"], "total_steps": r["steps"], "host_steps": st["host_steps"],
           "wall_s_end_to_end": wall, "output_ok": ok, "engine_error": r.get("engine_error", ""),
           "kernel_launches": st["kernel_launches"],
           "note": "reference CPU checker is quadratic in threads here (SURVEY F1: ~25 years extrapolated)"}
    if not args.no_c4:
        nb = 1 << 16
        r4, wall4 = _k1_run(gp.divergent_barrier_gen(nb, 1024, 0), "c4.cu", ws, rank, dev, shared)
        st4 = r4["stats"]
        stuck = [s for s in r4["stuck_reports"] if s["kind"] == "barrier"]
        # closed form: blocks b % 3 == 1 are all-odd (no deadlock), b % 3 == 0
        # all-even; b % 3 == 2 mixes parities -> deadlocked
        import numpy as np
        i = np.arange(nb * 1024, dtype=np.int64).reshape(nb, 1024)
        b = np.arange(nb, dtype=np.int64)[:, None]
        v = np.where(b % 3 == 0, 2 * i, np.where(b % 3 == 1, 2 * i + 1, (i * 3 + b) % 7))
        odd = (v % 2) == 1
        mixed = odd.any(1) & ~odd.all(1)
        exp_bids = np.nonzero(mixed)[0].tolist()
        got_bids = [s["bid"] for s in stuck]
        ok4 = r4["exit"] == 3 and got_bids == exp_bids and all(
            s["waiting"] == np.nonzero(odd[s["bid"]])[0].tolist() for s in stuck[:64])
        out["c4"] = {"workload": "C4: divergent-barrier deadlock sweep, 2^16 blocks x 1024 threads",
                     "deadlocks_ok": bool(ok4),
                     "thread_steps_per_s": st4["device_steps"] / (max(st4["grid_ms"], 1e-6) / 1e3),
                     "grid_ms": st4["grid_ms"], "device_steps": st4["device_steps"],
                     "barrier_rules": st4["barrier_rules"], "deadlocked_blocks": len(stuck),
                     "wall_s_end_to_end": wall4, "exit": r4["exit"],
                     "engine_error": r4.get("engine_error", ""), "kernel_launches": st4["kernel_launches"]}
    return out if rank == 0 else None


def run_e2e(args, torch, race, _abi):
    """Same metric through the host-buffer C-ABI call (H2D + D2H in the timed region)."""
    nb = args.e2e_blocks
    ev, bs = race.gen_c3(0, nb)
    hev = torch.empty(ev.shape, dtype=torch.int32, pin_memory=True)
    hev.copy_(ev)
    hbs = bs.cpu().numpy().astype("uint64")
    del ev, bs
    torch.cuda.empty_cache()
    lib = _abi.load()
    t = _abi.Trace(hev.data_ptr(), hbs.ctypes.data, hev.shape[0], nb, EVENTS_PER_BLOCK, 1, 0,
                   _abi.C3_SHMEM, 1)
    cap = nb * EVENTS_PER_BLOCK // 8
    import numpy as np
    tri = torch.empty((cap, 3), dtype=torch.int32, pin_memory=True)
    lf = np.zeros(_abi.MAX_LINES, dtype=np.uint64)
    n = ctypes.c_uint64(0)
    st = ctypes.c_uint32(0)

    def call():
        _abi.check(lib.mckg_detect_shared_host(ctypes.byref(t), ctypes.c_void_p(tri.data_ptr()),
                                               cap, ctypes.byref(n), lf.ctypes.data,
                                               ctypes.byref(st)), "mckg_detect_shared_host")

    call()
    steps = max(3, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = (time.perf_counter() - t0) / steps
    h2d = hev.numel() * 4 + hbs.nbytes
    d2h = int(n.value) * 12 + _abi.MAX_LINES * 8 + 8 + 4
    return {"value": nb * EVENTS_PER_BLOCK / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "api": "mckg_detect_shared_host (pinned host trace, chunked H2D overlapped with K2)",
            "events": nb * EVENTS_PER_BLOCK}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--blocks", type=int, default=FULL_BLOCKS)
    ap.add_argument("--e2e-blocks", type=int, default=FULL_BLOCKS)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="--impl reference: CPU seconds per step")
    ap.add_argument("--cpu-blocks", type=int, default=0,
                    help="blocks the cpu_baseline / parity leg replays (default: all of them)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dump", default="", help="directory: each rank saves its C3/C5 result sets (tests)")
    ap.add_argument("--no-k1", action="store_true")
    ap.add_argument("--k1-racy", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the K1 C4 deadlock-sweep leg")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--c5-blocks", type=int, default=0,
                    help="C5 blocks in total (default 2^17 per GPU: BASELINE configs[4] is 2^20 blocks = 2^32 events over 8 GPUs)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
