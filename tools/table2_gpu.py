"""Run the binary two-array recurrence on the GPU to convergence for l = lo..hi and compare the
certified bound with the paper's Table 2 ("rounded down to their 6th decimal
place").

  python tools/table2_gpu.py --lo 9 --hi 17 --dtype f64 > table2.jsonl
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TABLE2 = {}
for line in open(os.path.join(ROOT, "tests", "golden", "table2.txt")):
    if line.startswith("#") or not line.strip():
        continue
    f = line.split()
    TABLE2[int(f[0])] = (float(f[2]), int(f[3]))


def floor6(x):
    return math.floor(x * 1e6 + 1e-6) / 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lo", type=int, default=9)
    ap.add_argument("--hi", type=int, default=17)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--every", type=int, default=20)
    ap.add_argument("--max-sweeps", type=int, default=3000)
    ap.add_argument("--offsets", action="store_true",
                    help="integer-offset storage (offset_policy = 1, DESIGN.md reading R23)")
    args = ap.parse_args()
    import torch
    from paper_2407_10925_b200 import Lcsb
    for ell in range(args.lo, args.hi + 1):
        h = Lcsb(2, 2, ell, dtype=args.dtype, offset_policy=1 if args.offsets else 0)
        h.ready(wait=True)
        t0 = time.perf_counter()
        last = -1.0
        hist = []
        while h.sweeps_done < args.max_sweeps:
            h.sweep(args.every)
            b = h.bound()
            hist.append((b.sweeps_done, b.best_bound))
            if b.best_bound - last < 1e-10 and b.best_bound > 0:
                break
            last = b.best_bound
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        paper, line = TABLE2[ell]
        print(json.dumps({"ell": ell, "dtype": args.dtype, "sweeps": h.sweeps_done,
                          "best_bound": b.best_bound, "best_sweep": b.best_sweep,
                          "bound_at_Rmax": b.bound_at_Rmax, "bound_at_Rmin": b.bound_at_Rmin,
                          "floor6": floor6(b.best_bound), "paper": paper,
                          "paper_line": f"PAPER.md:{line}",
                          "match": floor6(b.best_bound) == paper, "seconds": dt,
                          "offsets": bool(args.offsets),
                          "kernel": h.kernel_in_use}), flush=True)
        h.destroy()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
