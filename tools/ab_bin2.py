"""A/B timing of the bin2 sweep variants (LCSB_BIN2_VARIANT) on one workload.

  python tools/ab_bin2.py --ell 17 --dtype f32 --sweeps 20
Each variant runs in a fresh handle; times the sweep with CUDA events; checks that every variant
produces the same sampled entries after the run.
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
    ap.add_argument("--variants", default="0,5,1,2,3,4")
    ap.add_argument("--shards", default="1", help="comma list of virtual shard counts")
    ap.add_argument("--warm", type=int, default=3, help="untimed sweeps first (graph capture)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2407_10925_b200 import Lcsb
    from seeded_inputs import splitmix64_indices
    idx = splitmix64_indices(7, 1 << 16, 1 << (2 * args.ell))
    ref = None
    esize = 4 if args.dtype == "f32" else 8
    runs = [(int(v), int(p)) for v in args.variants.split(",") for p in args.shards.split(",")]
    for v, p in runs:
        os.environ["LCSB_BIN2_VARIANT"] = str(v)
        h = Lcsb(2, 2, args.ell, dtype=args.dtype, shards=p, virtual_shards=p > 1)
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
            same = bool(np.array_equal(ref, vals))
        gbs = 2 * h.stored_states * esize / (ms / 1e3) / 1e9
        print(json.dumps({"variant": v, "shards": p, "ell": args.ell, "dtype": args.dtype, "ms_per_sweep": ms,
                          "alg_GBps": gbs, "frac_of_6557": gbs / 6557.1, "same_as_first": same}),
              flush=True)
        h.destroy()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
