import sys, numpy as np
f = open(sys.argv[1], "rb")
nt = int(np.frombuffer(f.read(8), dtype=np.int64)[0])
tr = np.frombuffer(f.read(8 * 4 * nt), dtype=np.uint64).reshape(nt, 4).astype(np.float64)
info = np.frombuffer(f.read(8 * nt), dtype=np.int32).reshape(nt, 2)
ok = tr[:, 2] > 0
t0 = tr[ok, 0].min()
c0, c1, e = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
span = e[ok].max()
wait = c1 - c0
work = e - c1
print(f"selinv tasks {ok.sum()} span {span/1e3:.1f} ms; CTA time waiting-for-deps {wait[ok].sum()/1e3:.1f} ms, working {work[ok].sum()/1e3:.1f} ms")
for k, nm in enumerate(["inner", "last-off", "last-diag", "group"]):
    m = ok & (info[:, 1] == k)
    if m.sum():
        print(f"  {nm:9s} n={m.sum():8d} mean work {work[m].mean():7.1f} us  mean wait {wait[m].mean():8.1f} us  mean pairs {info[m,0].mean():.2f}")
# work by pair count (inner chunks) and concurrency over time
for p in sorted(set(info[ok & (info[:, 1] == 0), 0].tolist()))[:12]:
    m = ok & (info[:, 1] == 0) & (info[:, 0] == p)
    if m.sum() > 20:
        print(f"  inner pairs={p:3d} n={m.sum():7d} work {work[m].mean():6.1f} us")
ts = np.linspace(0, span, 11)
for t in ts:
    busy = ((c1 <= t) & (e > t) & ok).sum()
    waiting = ((c0 <= t) & (c1 > t) & ok).sum()
    print(f"  t={t/1e3:7.2f} ms working {busy:4d} waiting {waiting:4d} done {((e <= t) & ok).sum():8d}")
# critical-path replay (actual last finisher chain) when successor lists are present
rest = f.read()
if rest:
    ns = int(np.frombuffer(rest[:8], dtype=np.int64)[0])
    sp = np.frombuffer(rest[8:8 + 4 * (nt + 1)], dtype=np.int32)
    su = np.frombuffer(rest[8 + 4 * (nt + 1):8 + 4 * (nt + 1) + 4 * ns], dtype=np.int32)
    ij = np.frombuffer(rest[8 + 4 * (nt + 1) + 4 * ns:], dtype=np.int32).reshape(nt, 2)
    src = np.repeat(np.arange(nt), np.diff(sp))
    order = np.argsort(su, kind="stable")
    pp = np.searchsorted(su[order], np.arange(nt + 1))
    preds_of = lambda t: src[order[pp[t]:pp[t + 1]]]
    t = int(np.argmax(np.where(ok, e, -1)))
    chain = []
    while True:
        chain.append(t)
        pr = preds_of(t)
        if pr.size == 0:
            break
        t = int(pr[np.argmax(e[pr])])
    chain = chain[::-1]
    tot_work = sum(work[t] for t in chain)
    gaps = [c1[chain[k]] - e[chain[k - 1]] for k in range(1, len(chain))]
    print(f"last-finisher chain: {len(chain)} tasks, work {tot_work/1e3:.1f} ms, gaps {sum(gaps)/1e3:.1f} ms (mean gap {np.mean(gaps):.1f} us)")
    kinds = ["inner", "last-off", "last-diag", "group"]
    from collections import Counter
    kc, kw = Counter(), Counter()
    for t in chain:
        kc[kinds[info[t, 1]]] += 1
        kw[kinds[info[t, 1]]] += work[t]
    print("  by kind:", {k: (kc[k], round(kw[k] / 1e3, 1)) for k in kc})
    mid = len(chain) // 2
    for t in chain[mid:mid + 12]:
        print(f"   {kinds[info[t,1]]:9s} tile ({ij[t,0]},{ij[t,1]}) pairs {info[t,0]:3d} work {work[t]:6.1f} us gap-before {c1[t] - max(e[preds_of(t)]) if preds_of(t).size else 0:6.1f} us")
