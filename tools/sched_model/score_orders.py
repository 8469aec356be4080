import numpy as np, pickle, sys
from collections import deque, defaultdict
ell = int(sys.argv[1]); G = 444
items = np.load(f'/tmp/sched/items_{ell}.npy'); ends = pickle.load(open(f'/tmp/sched/ends_{ell}.pkl','rb'))
E = len(items)
def dram(order, carry=0):
    """GB read: each wave of G items loads its distinct pieces (16 KB) once; pieces loaded in the
    previous `carry` waves are still in L2"""
    tot = 0; hist = deque()
    for w0 in range(0, len(order), G):
        s = set()
        for e in order[w0:w0+G]:
            s.update(ends[e][0]); s.update(ends[e][1])
        prev = set().union(*hist) if hist else set()
        tot += len(s - prev)
        hist.append(s)
        if len(hist) > carry: hist.popleft()
    return tot * 16384 / 1e9
nat = list(range(E))
print("natural", [round(dram(nat, c), 2) for c in (0, 1, 2)])
# v2 schedule (as lcsb_api.cu quarter_schedule)
nslots = 1 + max(max(e[2], e[3]) for e in ends)
adj = defaultdict(list)
for i, e in enumerate(ends):
    adj[e[2]].append(i)
    if e[3] != e[2]: adj[e[3]].append(i)
def other(i, v): return ends[i][3] if ends[i][2] == v else ends[i][2]
col = [-1]*nslots; order = []
for s0 in range(nslots):
    if col[s0] >= 0: continue
    col[s0] = 0; q = deque([s0]); order.append(s0)
    while q:
        u = q.popleft()
        for i in adj[u]:
            w = other(i, u)
            if col[w] < 0: col[w] = 1-col[u]; order.append(w); q.append(w)
for p in range(16):
    flips = 0
    for v in range(nslots):
        same = diff = 0
        for i in adj[v]:
            w = other(i, v)
            if w == v: continue
            if col[w] == col[v]: same += 1
            else: diff += 1
        if same > diff: col[v] ^= 1; flips += 1
    if not flips: break
done = [False]*E; grouped = [False]*nslots; sched = []
def emit(v):
    grouped[v] = True
    for i in adj[v]:
        if not done[i]: done[i] = True; sched.append(i)
for v in order:
    if col[v] == 0:
        if not grouped[v]: emit(v)
    else:
        for i in adj[v]:
            w = other(i, v)
            if col[w] == 0 and not grouped[w]: emit(w)
sched += [i for i in range(E) if not done[i]]
print("v2", [round(dram(sched, c), 2) for c in (0, 1, 2)])
pickle.dump((sched,), open(f'/tmp/sched/v2_{ell}.pkl','wb'))
