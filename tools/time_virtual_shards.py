"""Time the sharded quarter table on P virtual shards of ONE GPU: the same sweep
kernel over one virtual address range per table, one launch per shard over its item list.
Shows what the sharding itself costs on one GPU (no NVLink involved).

  python tools/time_virtual_shards.py --ell 17 --shards 1 2 4 8
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
    ap.add_argument("--shards", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--sweeps", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_2407_10925_b200 import Lcsb
    for P in args.shards:
        kw = dict(shards=P, virtual_shards=True) if P > 1 else {}
        h = Lcsb(2, 2, args.ell, dtype=args.dtype, symmetry=2, **kw)
        h.ready(wait=True)
        h.sweep(3)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.sweep(args.sweeps)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / args.sweeps
        s.record()
        b = h.bound()
        e.record()
        torch.cuda.synchronize()
        tr = h.shard_traffic() if P > 1 else None
        print(json.dumps({"ell": args.ell, "shards": P, "kernel": h.kernel_in_use,
                          "ms_per_sweep": ms, "bound_ms": s.elapsed_time(e),
                          "state_updates_per_s": (1 << (2 * args.ell)) / (ms / 1e3),
                          "cross_shard_bytes_per_sweep": (tr[0] + tr[1]) if tr else 0,
                          "device_bytes": h.device_bytes}), flush=True)
        h.destroy()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
