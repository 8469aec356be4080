"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2407_10925_b200 import Lcsb
    runs = [
        dict(sigma=2, d=2, ell=8, dtype="f32"),                      # bin2 TMA / register
        dict(sigma=2, d=2, ell=12, dtype="f32"),                     # bin2 TMA M=6
        dict(sigma=2, d=2, ell=11, dtype="f64"),                     # bin2 TMA fp64 staged stores
        dict(sigma=2, d=2, ell=9, dtype="f32", shards=4, virtual_shards=True),
        dict(sigma=4, d=2, ell=4, dtype="f32", form="ks"),           # q4
        dict(sigma=3, d=3, ell=2, dtype="f64", form="ks"),           # small
        dict(sigma=3, d=3, ell=2, dtype="f64", form="ks", kernel="generic"),
        dict(sigma=5, d=2, ell=1, dtype="f64", form="ks"),           # generic runtime (sigma, d)
    ]
    for kw in runs:
        h = Lcsb(**kw)
        h.sweep(40)
        b = h.bound()
        t = h.table(0, 0, min(h.num_states, 1 << 12))
        g = h.table_gather(np.arange(0, h.num_states, max(1, h.num_states // 997), dtype=np.uint64))
        torch.cuda.synchronize()
        print(kw, h.kernel_in_use, f"{b.bound:.9f}", float(t.sum()), float(g.sum()), flush=True)
        h.destroy()
    print("sanitize driver done")


if __name__ == "__main__":
    main()
