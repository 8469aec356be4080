"""Time the quarter table's bound paths at one l (reading R25): per sweep, a plain sweep
and a tracking sweep; per bound, the one-pass bound, the D-only pass after a tracked sweep, and
the step "S sweeps + bound" done three ways -- sweep(S) + bound (one pass), sweep_ex(S, TRACK) +
bound (D pass), sweep_bound(S) (bound of iterate S-1, no pass).  CUDA events on torch's current
stream (the library's stream), after warm-up; one JSON line.
  python tools/time_tracking.py --ell 17 --dtype f32 --steps 3
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
    ap.add_argument("--sweeps", type=int, default=50)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_2407_10925_b200 import lcsb as L
    h = L.Lcsb(2, 2, args.ell, dtype=args.dtype, symmetry=2)
    h.ready(wait=True)
    h.sweep(4)
    torch.cuda.synchronize()

    def ev(fn, reps=args.reps):
        out = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            out.append(s.elapsed_time(e))
        return sorted(out)[len(out) // 2]

    res = {"ell": args.ell, "dtype": args.dtype}
    res["plain_sweep_ms"] = ev(lambda: h.sweep(10)) / 10
    res["tracked_sweep_ms"] = ev(lambda: [h.sweep_ex(1, 1) for _ in range(10)]) / 10
    h.sweep(1)
    res["one_pass_bound_ms"] = ev(h.bound)
    h.sweep_ex(1, 1)
    res["d_pass_bound_ms"] = ev(h.bound)
    S = args.sweeps
    res["step_sweep_bound_onepass_ms"] = ev(lambda: (h.sweep(S), h.bound()), 3)
    res["step_sweep_ex_dpass_ms"] = ev(lambda: (h.sweep_ex(S, 1), h.bound()), 3)
    res["step_sweep_bound_fused_ms"] = ev(lambda: h.sweep_bound(S), 3)
    res["bounds"] = [h.bound().bound]
    print(json.dumps(res))
    h.destroy()


if __name__ == "__main__":
    main()
