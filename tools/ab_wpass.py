"""Time lcsb_bound (R pass + W pass) for W-pass settings given by environment knobs.
  LCSB_WPASS_M=6 LCSB_WPASS_STAGES=1 python tools/ab_wpass.py --ell 17 --dtype f32"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ell", type=int, default=17)
    ap.add_argument("--dtype", default="f32")
    args = ap.parse_args()
    import torch
    from paper_2407_10925_b200 import Lcsb
    h = Lcsb(2, 2, args.ell, dtype=args.dtype)
    h.sweep(5)
    b0 = h.bound()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        b = h.bound()
    dt = (time.perf_counter() - t) / 3
    print(json.dumps({"M": os.environ.get("LCSB_WPASS_M"), "stages": os.environ.get(
        "LCSB_WPASS_STAGES"), "ell": args.ell, "dtype": args.dtype, "bound_ms": dt * 1e3,
        "bound": b.bound, "same": b.bound == b0.bound and b.E_at_Rmax == b0.E_at_Rmax}))


if __name__ == "__main__":
    main()
