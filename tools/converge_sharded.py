"""Run the binary two-array recurrence to convergence on the SHARDED half table (one process per
GPU under torchrun) -- the runs one B200 cannot hold:

  l = 18, fp64 storage (2 x 2^35 x 8 B = 550 GB: 4 GPUs) -> Table 2's 0.790668,
      the sixth digit fp32 storage misses (0.790656, results/r01_table2_gpu_f32_l18.jsonl);
  l = 19, fp32 storage (2 x 2^37 x 4 B = 1.1 TB: 8 GPUs) -> 0.791389, the paper's
      first external-memory point (183,431 s, "switch to external memory" PAPER.md:44).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/converge_sharded.py --ell 18 --dtype f64
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/converge_sharded.py --ell 19 --dtype f32

The bound is evaluated every --every sweeps until the best bound stops improving (as
tools/table2_gpu.py); rank 0 prints one JSON line per evaluation and a final one.  With
--transport host and LCSB_BENCH_DEVICE=0 the same script runs its ranks on one GPU (small l
only: a test of the path, not a measurement).
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAPER = {18: (0.790668, 73), 19: (0.791389, 74)}  # Table 2, "rounded down"


def floor6(x):
    return math.floor(x * 1e6 + 1e-6) / 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ell", type=int, default=18)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--every", type=int, default=20)
    ap.add_argument("--max-sweeps", type=int, default=600)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"])
    ap.add_argument("--offsets", type=int, default=0,
                    help="offset_policy (1: integer offsets, readings R23 / R26; fp32 drift 4-30x lower)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2407_10925_b200.dist import create_sharded
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LCSB_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    if args.transport == "host":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    h = create_sharded(args.ell, dtype=args.dtype, transport=args.transport,
                       offset_policy=args.offsets)
    t0 = time.perf_counter()
    last = -1.0
    while h.sweeps_done < args.max_sweeps:
        h.sweep(args.every)
        b = h.bound()  # collective
        if rank == 0:
            print(json.dumps({"ell": args.ell, "dtype": args.dtype, "shards": h.num_shards,
                              "sweeps": b.sweeps_done, "bound": b.bound,
                              "best_bound": b.best_bound,
                              "seconds": time.perf_counter() - t0}), flush=True)
        if b.best_bound - last < 1e-10 and b.best_bound > 0:
            break
        last = b.best_bound
    if rank == 0:
        paper, line = PAPER.get(args.ell, (None, None))
        print(json.dumps({"final": True, "ell": args.ell, "dtype": args.dtype,
                          "shards": h.num_shards, "sweeps": b.sweeps_done,
                          "best_bound": b.best_bound, "best_sweep": b.best_sweep,
                          "floor6": floor6(b.best_bound), "paper": paper,
                          "paper_line": f"PAPER.md:{line}" if line else None,
                          "match": floor6(b.best_bound) == paper if paper else None,
                          "seconds": time.perf_counter() - t0}), flush=True)
    h.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
