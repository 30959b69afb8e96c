"""Analyze a PINLA_TRACE_SOLVE dump of one solve launch (slot 0): the
forward/backward tile-row chains, handoff latency link-producer -> row task."""
import sys
from collections import defaultdict
import numpy as np

f = open(sys.argv[1], "rb")
nb, S, nT = np.frombuffer(f.read(24), dtype=np.int64)
tk = np.frombuffer(f.read(16 * nb), dtype=np.int32).reshape(nb, 4)
tr = np.frombuffer(f.read(8 * 8 * nb * S), dtype=np.uint64).reshape(nb * S, 8).astype(np.float64)
trow = np.frombuffer(f.read(4 * nT), dtype=np.int32)
tcol = np.frombuffer(f.read(4 * nT), dtype=np.int32)
inst = np.arange(nb) * S  # slot 0 instances
T = tr[inst]
ok = T[:, 2] > 0
t0 = T[ok, 0].min()
cl, rd, en = (T[:, 0] - t0) / 1e3, (T[:, 4] - t0) / 1e3, (T[:, 5] - t0) / 1e3
ew, es, lt = (T[:, 1] - t0) / 1e3, (T[:, 2] - t0) / 1e3, (T[:, 3] - t0) / 1e3
print(f"tasks {ok.sum()} span {en[ok].max():.1f} us")
for ty, name in ((0, "fwd row"), (1, "fwd prod"), (2, "bwd col"), (3, "bwd prod")):
    m = ok & (tk[:, 0] == ty)
    if m.any():
        print(f"  {name:8s} n={m.sum():7d} claim->ready {np.median(rd[m]-cl[m]):7.2f} us  ready->end {np.median(en[m]-rd[m]):6.2f} us (median)")
# row form: newest off-diagonal of each row
NT = trow.max() + 1
rows = defaultdict(list)
for t in range(nT):
    if trow[t] != tcol[t]:
        rows[trow[t]].append((tcol[t], t))
cols = defaultdict(list)
for t in range(nT):
    if trow[t] != tcol[t]:
        cols[tcol[t]].append((trow[t], t))
row_task = {int(tk[i, 2]): i for i in range(nb) if tk[i, 0] == 0}
col_task = {int(tk[i, 2]): i for i in range(nb) if tk[i, 0] == 2}
prod_task = {int(tk[i, 2]): i for i in range(nb) if tk[i, 0] == 1}
bprod_task = {int(tk[i, 2]): i for i in range(nb) if tk[i, 0] == 3}
hand, comp, late_gap = [], [], []
for I in range(NT):
    r = sorted(rows.get(I, []))
    if not r:
        continue
    link = r[-1][0]
    a, b = row_task[I], row_task[link]
    hand.append(rd[a] - en[b])
    comp.append(en[a] - rd[a])
hand, comp = np.array(hand), np.array(comp)
ph = defaultdict(list)
for I in range(NT):
    r = sorted(rows.get(I, []))
    if len(r) < 3:
        continue
    a, b = row_task[I], row_task[r[-1][0]]
    for nm, v in (("early-wait done", ew[a]), ("early sum done", es[a]), ("late done", lt[a]), ("ready", rd[a]), ("end", en[a])):
        ph[nm].append(v - rd[b])
print("row task phase times relative to the link row's READY time (median us):",
      {k: round(float(np.median(v)), 2) for k, v in ph.items()})
print(f"fwd chain: link end -> row ready: median {np.median(hand):.2f} us, p90 {np.percentile(hand,90):.2f}; row ready -> end {np.median(comp):.2f} us")
if late_gap:
    lg = np.array(late_gap)
    print(f"  late partial end - link end: median {np.median(lg):.2f} us (positive = late partial arrives after the link)")
hb, cb = [], []
for J in range(NT):
    c = sorted(cols.get(J, []))
    if not c:
        continue
    link = c[0][0]
    a, b = col_task[J], col_task[link]
    hb.append(rd[a] - en[b])
    cb.append(en[a] - rd[a])
print(f"bwd chain: link end -> col ready: median {np.median(hb):.2f} us; ready -> end {np.median(cb):.2f} us")
fr = [en[row_task[I]] for I in range(NT) if I in row_task]
bc = [en[col_task[J]] for J in range(NT) if J in col_task]
print(f"forward sweep ends at {max(fr):.1f} us; backward sweep {max(bc) - max(fr):.1f} us after; per tile row fwd {max(fr)/NT:.2f} us")
