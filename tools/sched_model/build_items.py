"""Offline model of the folded-table sweep's DRAM reads for an item order ("L2
item schedule"): each wave of G consecutive items loads every distinct 16 KB block-quarter it
touches once.  Step 1: the items (tile pairs) and the stored pieces of their two windows.
  python tools/sched_model/build_items.py 17     (writes /tmp/sched/items_17.npy, ends_17.pkl)
then score_orders.py (natural and v2 orders) and greedy_waves.py (the v4 re-cut)."""
import numpy as np, sys, time
ell, K, M, G = int(sys.argv[1]), 7, 6, 444
L = 2*ell; lmask = (1<<L)-1; q1 = 1<<(L-2)
A = 0xAAAAAAAAAAAAAAAA & lmask; B = 0x5555555555555555 & lmask
T = 1<<(2*M); PL = 2*(ell-K); pm = (1<<PL)-1; tailm = (1<<(PL-2))-1
def ps(v): return ((v & 0xAAAAAAAAAAAAAAAA) >> 1) | ((v & 0x5555555555555555) << 1)
def image(b, g):
    if (b >> (PL-2)) & 1: return ps(~b & pm) & pm
    if g == 1: return ps(b) & pm
    if g == 3: return b ^ tailm
    return ps(b ^ tailm) & pm
nb = 1 << (PL-1)
canon = np.empty(nb, np.int64); how = np.empty(nb, np.int8)
for b in range(nb):
    c, g0 = b, 0
    for g in ((2,) if (b >> (PL-2)) & 1 else (1,2,3)):
        im = image(b, g)
        if im < c: c, g0 = im, g
    canon[b] = c; how[b] = g0
slots = {c: i for i, c in enumerate(sorted(set(canon.tolist())))}
slot = np.array([slots[c] for c in canon.tolist()], np.int64)
kmask = (1<<(2*K))-1
def win(x): return (x & A) | ((x & B & ~q1) << 2)
def pieces(w):
    """stored (slot, quarter) pieces of the logical window starting at half-table index w"""
    bl = w >> (2*K); e = w & kmask; s = slot[bl]; m = how[bl]
    if m == 0: offs = [e, e + T]
    elif m == 3: st = (~e & kmask) & ~(2*T-1); offs = [st, st + T]
    else:
        f = ps(e) & kmask if m == 1 else ps(~e & kmask) & kmask
        st = (f & ~(4*T-1)) | (f & T); offs = [st, st + 2*T]
    return [(int(s) << 2) | (o // T) % 4 for o in offs]
ntiles = 1 << (2*(ell-1-M))
items = []; ends = []
for tau in range(ntiles):
    x0 = q1 + tau*T; p0 = ps(~x0 & lmask) & ~(T-1)
    if ((p0 - q1) >> (2*M)) < tau: continue
    items.append(tau); ends.append((pieces(win(x0)), pieces(win(p0)), int(slot[win(x0) >> (2*K)]), int(slot[win(p0) >> (2*K)])))
np.save(f'/tmp/sched/items_{ell}.npy', np.array(items))
import pickle; pickle.dump(ends, open(f'/tmp/sched/ends_{ell}.pkl','wb'))
print("items", len(items), "stored blocks", len(slots))
