import numpy as np, pickle, sys
from collections import defaultdict, deque
ell = int(sys.argv[1]); G = 444
items = np.load(f'/tmp/sched/items_{ell}.npy'); ends = pickle.load(open(f'/tmp/sched/ends_{ell}.pkl','rb'))
(v2,) = pickle.load(open(f'/tmp/sched/v2_{ell}.pkl','rb'))
E = len(items)
exec(open('/tmp/sched/score.py').read().split('nat = list')[0].split('E = len(items)')[1])  # dram()
pcs = [list(set(e[0]) | set(e[1])) for e in ends]
inv = defaultdict(list)
for i, p in enumerate(pcs):
    for q in p: inv[q].append(i)
done = np.zeros(E, bool); order = []; seed_ptr = 0
while len(order) < E:
    # seed: next unscheduled item in v2 order
    while done[v2[seed_ptr]]: seed_ptr += 1
    hot = set(); score = {}; buckets = defaultdict(set); cnt = 0
    def add(i):
        global cnt
        done[i] = True; order.append(i); cnt += 1
        sc = score.pop(i, None)
        if sc is not None: buckets[sc].discard(i)
        for q in pcs[i]:
            if q in hot: continue
            hot.add(q)
            for j in inv[q]:
                if done[j]: continue
                s0 = score.get(j, 0)
                if s0: buckets[s0].discard(j)
                score[j] = s0 + 1; buckets[s0 + 1].add(j)
    add(v2[seed_ptr])
    while cnt < G and len(order) < E:
        pick = None
        for s in (4, 3, 2, 1):
            if buckets[s]:
                pick = buckets[s].pop(); break
        if pick is None:
            while seed_ptr < E and done[v2[seed_ptr]]: seed_ptr += 1
            if seed_ptr >= E: break
            pick = v2[seed_ptr]
        score.pop(pick, None)
        add(pick)
print("greedy", [round(dram(order, c), 2) for c in (0, 1, 2)])
pickle.dump(order, open(f'/tmp/sched/greedy_{ell}.pkl','wb'))
