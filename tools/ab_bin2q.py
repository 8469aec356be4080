"""A/B timing of the quarter-table sweep variants (LCSB_BIN2Q_VARIANT) against the half table.

  python tools/ab_bin2q.py --ell 17 --dtype f32 --sweeps 20 --variants 0,1,2,3
Each variant runs in a fresh handle; the sweep is timed with CUDA events; every variant must
give the same sampled entries as the half table.  alg_GBps counts the layout's compulsory bytes
(2 x stored: read once, write once); moved_GBps the bytes the kernel requests (half table: 2 x
stored; quarter table: 3 x stored -- every stored block is loaded once per logical image; with
the L2 item schedule part of the second loads hit L2, so this can exceed the DRAM peak).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ell", type=int, default=17)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--sweeps", type=int, default=20)
    ap.add_argument("--variants", default="0,1,2,3,4,5,6,7,8,9,10")
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--peak", type=float, default=None)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2407_10925_b200 import Lcsb
    from seeded_inputs import splitmix64_indices
    peak = args.peak
    if peak is None:
        try:
            peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
                os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            peak = 6650.0
    idx = splitmix64_indices(7, 1 << 16, 1 << (2 * args.ell))
    esize = 4 if args.dtype == "f32" else 8
    ref = None
    for v in ["half"] + args.variants.split(","):
        if v == "half":
            os.environ.pop("LCSB_BIN2Q_VARIANT", None)
            h = Lcsb(2, 2, args.ell, dtype=args.dtype, symmetry=1)
            moved = 2
        else:
            os.environ["LCSB_BIN2Q_VARIANT"] = v
            try:
                h = Lcsb(2, 2, args.ell, dtype=args.dtype, symmetry=2)
            except Exception as e:  # variant does not fit this l / block size
                print(json.dumps({"variant": v, "error": str(e)}), flush=True)
                continue
            moved = 3
        h.sweep(args.warm)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.sweep(args.sweeps)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / args.sweeps
        vals = h.table_gather(idx)
        same = None
        if ref is None:
            ref = vals
        else:
            same = bool(np.array_equal(ref, vals)) if args.dtype == "f32" else \
                bool(np.allclose(ref, vals, rtol=1e-12, atol=0))
        alg = 2 * h.stored_states * esize / (ms / 1e3) / 1e9
        mov = moved * h.stored_states * esize / (ms / 1e3) / 1e9
        print(json.dumps({"variant": v, "ell": args.ell, "dtype": args.dtype,
                          "ms_per_sweep": ms, "state_updates_per_s": h.num_states / (ms / 1e3),
                          "alg_GBps": alg, "moved_GBps": mov, "moved_frac": mov / peak,
                          "same_as_half": same}), flush=True)
        h.destroy()
        torch.cuda.empty_cache()
    os.environ.pop("LCSB_BIN2Q_VARIANT", None)


if __name__ == "__main__":
    main()
