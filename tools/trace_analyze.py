"""Analyze a PINLA_TRACE dump of one factor launch."""
import sys
import numpy as np
f = open(sys.argv[1], "rb")
nb, S = np.frombuffer(f.read(16), dtype=np.int64)
tk = np.frombuffer(f.read(16 * nb), dtype=np.int32).reshape(nb, 4)
tr = np.frombuffer(f.read(8 * 4 * nb * S), dtype=np.uint64).reshape(nb * S, 4).astype(np.float64)
npairs = np.frombuffer(f.read(8 * nb), dtype=np.int64)
ok = tr[:, 2] > 0
t0 = tr[ok, 0].min()
claim = (tr[:, 0] - t0) / 1e3
end = (tr[:, 2] - t0) / 1e3
dur = end - claim
span = end[ok].max()
print(f"tasks {ok.sum()} span {span:.1f} us; sum of task durations {dur[ok].sum()/1e3:.1f} ms over {int(tr[ok,3].max())+1} SMs")
typ = np.repeat(tk[:, 0], S)
isdiag = np.repeat(npairs >= 1000, S)
for name, m in (("partial", typ == 1), ("diag", (typ == 0) & isdiag), ("offdiag", (typ == 0) & ~isdiag)):
    m = m & ok
    print(f"{name:8s} n={m.sum():6d} mean dur {dur[m].mean():8.1f} us  max {dur[m].max():8.1f}  total {dur[m].sum()/1e3:8.1f} ms")
# timeline: how many tasks in flight over time
ts = np.linspace(0, span, 20)
for t in ts:
    inflight = ((claim <= t) & (end > t) & ok).sum()
    done = ((end <= t) & ok).sum()
    print(f"t={t:8.1f}us inflight {inflight:4d} done {done:6d}")
# last finishing tasks
idx = np.argsort(-end)[:15]
for i in idx:
    b = i // S
    print(f"task {i} type {tk[b,0]} id {tk[b,2]} level {tk[b,3]} npairs {npairs[b]} claim {claim[i]:.1f} end {end[i]:.1f} dur {dur[i]:.1f}")
