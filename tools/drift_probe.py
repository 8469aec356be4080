"""fp32 storage drift with and without integer offsets (readings R23 / R26), against fp64 storage,
on one GPU: the bound after each checkpoint of sweeps for fp32, fp32 + offsets and fp64.

  python tools/drift_probe.py --sigma 4 --d 2 --ell 8 --form ks --checkpoints 100,300
Prints one JSON line per (storage, checkpoint): bound at R_max / R_min and the relative error of
the fp32 runs against the fp64 run at the same sweep count.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sigma", type=int, default=4)
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--ell", type=int, default=8)
    ap.add_argument("--form", default="ks")
    ap.add_argument("--checkpoints", default="100,300")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    from paper_2407_10925_b200 import Lcsb
    cps = [int(c) for c in args.checkpoints.split(",")]
    runs = {}
    for name, dtype, ofs in (("f64", "f64", 0), ("f32", "f32", 0), ("f32_offsets", "f32", 1)):
        h = Lcsb(args.sigma, args.d, args.ell, dtype=dtype, form=args.form, offset_policy=ofs)
        h.ready(wait=True)
        done, out = 0, {}
        for c in cps:
            h.sweep(c - done)
            done = c
            b = h.bound()
            out[c] = (b.bound_at_Rmax, b.bound_at_Rmin, h.kernel_in_use)
        h.destroy()
        runs[name] = out
    for name, out in runs.items():
        for c, (bmax, bmin, kern) in out.items():
            ref = runs["f64"][c][0]
            print(json.dumps({"tag": args.tag, "sigma": args.sigma, "d": args.d, "ell": args.ell,
                              "form": args.form, "storage": name, "kernel": kern, "sweeps": c,
                              "bound_at_Rmax": bmax, "bound_at_Rmin": bmin,
                              "rel_err_vs_f64": abs(bmax - ref) / abs(ref) if ref else None}),
                  flush=True)


if __name__ == "__main__":
    main()
