"""Minimal driver for ncu captures: one handle of a bench workload, a few sweeps and one bound.

  python tools/ncu_driver.py --workload config4 --sweeps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import WORKLOADS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config4", choices=sorted(WORKLOADS))
    ap.add_argument("--sweeps", type=int, default=3)
    ap.add_argument("--ell", type=int, default=None, help="override l (same kernel, smaller table)")
    ap.add_argument("--symmetry", type=int, default=-1, help="-1 auto, 1 half, 2 quarter table")
    ap.add_argument("--tracked", action="store_true",
                    help="the last two sweeps are tracking sweeps, then the D-only bound pass")
    args = ap.parse_args()
    import torch
    from paper_2407_10925_b200 import Lcsb
    w = dict(WORKLOADS[args.workload])
    if args.ell:
        w["ell"] = args.ell
    h = Lcsb(w["sigma"], w["d"], w["ell"], dtype=w["dtype"], form=w["form"],
             symmetry=args.symmetry)
    h.ready(wait=True)  # the quarter table's item schedule (host thread) before the first sweep
    if args.tracked:
        h.sweep_ex(args.sweeps, 3)
    else:
        h.sweep(args.sweeps)
    b = h.bound()
    torch.cuda.synchronize()
    print(f"{args.workload} l={w['ell']} sweeps={args.sweeps} kernel={h.kernel_in_use} "
          f"bound={b.bound:.9f}")
    h.destroy()


if __name__ == "__main__":
    main()
