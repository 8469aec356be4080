"""Why the bound is slower inside the bench loop than alone (round 2): times lcsb_bound at l = 17
after 4 sweeps, after 50 back-to-back sweeps (the bench step), and after 50 sweeps plus 1 s idle.
Measured: 10.87 / 13.31 / 10.89 ms -- the sustained sweep load runs under sw_power_cap (SM clock
~1700 of 1965 MHz) and the latency-bound bound pass slows with the SM clock (the bandwidth-bound
sweep only 5.12 -> 5.40 ms).  ncu (serialised launches, no power cap) gives 10.83 ms at both points.
"""
import json, statistics, sys, time
sys.path.insert(0, ".")
import torch
from paper_2407_10925_b200 import Lcsb
h = Lcsb(2, 2, 17, dtype="f32")
h.ready(wait=True)
s = torch.cuda.current_stream()
def ev():
    return torch.cuda.Event(enable_timing=True)
res = {}
for S in (4, 50):
    t = {"b1": [], "b2": [], "sw": []}
    for rep in range(5):
        h.reset()
        a, b, c, d = ev(), ev(), ev(), ev()
        a.record(s); h.sweep(S); b.record(s)
        h.bound(); c.record(s)
        h.bound(); d.record(s)
        torch.cuda.synchronize()
        t["sw"].append(a.elapsed_time(b) / S); t["b1"].append(b.elapsed_time(c)); t["b2"].append(c.elapsed_time(d))
    res[S] = {k: round(statistics.median(v), 3) for k, v in t.items()}
t = []
for rep in range(5):
    h.reset(); h.sweep(50); torch.cuda.synchronize(); time.sleep(1.0)
    a, b = ev(), ev()
    a.record(s); h.bound(); b.record(s); torch.cuda.synchronize()
    t.append(a.elapsed_time(b))
res["50_then_idle_1s"] = round(statistics.median(t), 3)
print(json.dumps(res))
