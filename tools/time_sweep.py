"""Time the sweep of one (sigma, d, l) handle (A/B of the LCSB_* knobs, one process per setting).

  LCSB_Q4_FLAGS=0 python tools/time_sweep.py --sigma 4 --d 2 --ell 8 --dtype f32
Prints one JSON line: ms per sweep (CUDA events around --sweeps sweeps after --warm), the kernel
in use, and a hash of 2^16 seeded entries of the newest table so settings can be checked equal.
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigma", type=int, default=4)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--ell", type=int, default=8)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--form", default="auto")
    ap.add_argument("--sweeps", type=int, default=20)
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default="")
    ap.add_argument("--offsets", action="store_true", help="offset_policy = 1 (R23 / R26)")
    ap.add_argument("--residual", action="store_true",
                    help="offsets + lcsb_rebase after the warm-up: time the residual sweep (R24)")
    args = ap.parse_args()
    import torch
    from paper_2407_10925_b200 import Lcsb
    from seeded_inputs import splitmix64_indices
    h = Lcsb(args.sigma, args.d, args.ell, dtype=args.dtype, form=args.form,
             offset_policy=1 if (args.residual or args.offsets) else 0)
    h.ready(wait=True)
    h.sweep(args.warm)
    if args.residual:
        h.rebase()
        h.sweep(1)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.sweep(args.sweeps)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / args.sweeps)
    b = h.bound()
    torch.cuda.synchronize()
    bt = []
    for _ in range(args.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        b = h.bound()  # R reduction + W pass + E (host read of the result included)
        e.record()
        torch.cuda.synchronize()
        bt.append(s.elapsed_time(e))
    idx = splitmix64_indices(7, 1 << 16, h.num_states)
    digest = hashlib.sha1(h.table_gather(idx).tobytes()).hexdigest()[:16]
    print(json.dumps({"tag": args.tag, "sigma": args.sigma, "d": args.d, "ell": args.ell,
                      "dtype": args.dtype, "kernel": h.kernel_in_use,
                      "ms_per_sweep": min(times), "ms_all": times,
                      "state_updates_per_s": h.num_states / (min(times) / 1e3),
                      "bound_ms": min(bt), "bound": b.bound, "sample_sha1": digest}),
          flush=True)
    h.destroy()


if __name__ == "__main__":
    main()
