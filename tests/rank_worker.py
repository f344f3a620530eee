"""Worker for tests/test_gpu_rank_sharded.py (launched by torchrun): every
rank runs the same programs with its block range of each grid
(run_source(rank=, world=)); memory and reports are combined over the host
transport (gloo) or NCCL.  Rank 0 writes the projected results as JSON."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def main():
    import torch
    import torch.distributed as dist
    from paper_1211_6193_b200 import checker
    from program_corpus import corpus, project
    out_path, transport, names = sys.argv[1], sys.argv[2], sys.argv[3].split(",")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    dev = 0 if transport == "host" else rank
    torch.cuda.set_device(dev)
    kw = dict(rank=rank, world=world, device=dev)
    if transport == "host":
        kw["allgather"] = checker.torch_allgather()
    else:
        obj = [checker.comm_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        kw["comm"] = obj[0]
    progs = {n: (f, s) for n, f, s in corpus()}
    res = {}
    for n in names:
        fname, src = progs[n]
        r = checker.run_source(src, filename=fname, **kw)
        res[n] = dict(project(r), engine_error=r.get("engine_error", ""))
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
