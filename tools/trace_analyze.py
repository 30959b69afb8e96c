"""Analyze a PINLA_TRACE dump of one factor launch (chunk tasks)."""
import sys
import numpy as np
f = open(sys.argv[1], "rb")
nb, S = np.frombuffer(f.read(16), dtype=np.int64)
tk = np.frombuffer(f.read(16 * nb), dtype=np.int32).reshape(nb, 4)
tr8 = np.frombuffer(f.read(8 * 8 * nb * S), dtype=np.uint64).reshape(nb * S, 8).astype(np.float64)
tr = tr8[:, :4]
code = np.frombuffer(f.read(8 * nb), dtype=np.int64)
ok = tr[:, 2] > 0
t0 = tr[ok, 0].min()
claim = (tr[:, 0] - t0) / 1e3
end = (tr[:, 2] - t0) / 1e3
dur = end - claim
span = end[ok].max()
print(f"tasks {ok.sum()} span {span:.1f} us; sum of task durations {dur[ok].sum()/1e3:.1f} ms; avg concurrency {dur[ok].sum()/span:.1f}")
# task instance i -> base = i % nb (instances laid out slot-major)
base = np.arange(nb * S) % nb
pairs = code[base] % 1000
diag = (code[base] // 1000) % 10 == 1
last = code[base] >= 10000
for name, m in (("last-diag", last & diag), ("last-off", last & ~diag), ("inner", ~last)):
    m = m & ok
    if m.sum() == 0:
        continue
    print(f"{name:9s} n={m.sum():6d} mean dur {dur[m].mean():7.1f} us  mean pairs {pairs[m].mean():5.2f}  total {dur[m].sum()/1e3:7.1f} ms")
for p in range(0, 17):
    m = ok & (pairs == p) & ~diag
    if m.sum() > 50:
        print(f"  offdiag pairs={p:2d} n={m.sum():6d} mean {dur[m].mean():6.1f} us  median {np.median(dur[m]):6.1f}")
# sub-phases (medians, us): pop (claim + dependency wait), setup (C init),
# pairs, finalize math, stores, completion (fence + successors)
pop_s, set_s, fin_s, sto_s = (tr8[:, 4] - t0) / 1e3, (tr8[:, 5] - t0) / 1e3, (tr8[:, 6] - t0) / 1e3, (tr8[:, 7] - t0) / 1e3
mid_s = (tr[:, 1] - t0) / 1e3
for name, m in (("last-diag", last & diag), ("last-off", last & ~diag), ("inner", ~last)):
    m = m & ok & (tr8[:, 5] > 0)
    if m.sum() == 0:
        continue
    d = {"pop": np.median(claim[m] - pop_s[m]), "setup": np.median(set_s[m] - claim[m]),
         "pairs": np.median(mid_s[m] - set_s[m])}
    if name != "inner":
        d["fin_math"] = np.median(fin_s[m] - mid_s[m])
        d["stores"] = np.median(sto_s[m] - fin_s[m])
        d["complete"] = np.median(end[m] - sto_s[m])
    else:
        d["store+complete"] = np.median(end[m] - mid_s[m])
    print(f"  {name:9s} phases (median us):", {k: round(float(v), 2) for k, v in d.items()})
ts = np.linspace(0, span, 12)
for t in ts:
    print(f"t={t:8.1f}us inflight {((claim <= t) & (end > t) & ok).sum():4d} done {((end <= t) & ok).sum():6d}")
mid = (tr[:, 1] - t0) / 1e3
m = ok & last & diag & (tr[:, 1] > 0)
print("last-diag: pre-finalize part mean", np.mean(mid[m] - claim[m]), "finalize mean", np.mean(end[m] - mid[m]))
print("last-diag dur percentiles", np.percentile(dur[m], [5, 25, 50, 75, 95, 99]))
m2 = ok & last & ~diag & (tr[:, 1] > 0)
print("last-off: pre mean", np.mean(mid[m2] - claim[m2]), "finalize mean", np.mean(end[m2] - mid[m2]))
# critical path replay with measured durations (slot 0 instances)
rest = f.read()
if rest:
    ns = np.frombuffer(rest[:8], dtype=np.int64)[0]
    sp = np.frombuffer(rest[8:8 + 4 * (nb + 1)], dtype=np.int32)
    su = np.frombuffer(rest[8 + 4 * (nb + 1):8 + 4 * (nb + 1) + 4 * ns], dtype=np.int32)
    # predecessor lists from successor lists
    preds = [[] for _ in range(nb)]
    for t in range(nb):
        for u in su[sp[t]:sp[t + 1]]:
            preds[u].append(t)
    for slot in range(min(S, 2)):
        d = dur[slot * nb:(slot + 1) * nb]
        EF = np.zeros(nb)
        best = np.full(nb, -1)
        # tasks are topologically ordered? compute via Kahn order using ndeps
        indeg = np.array([len(p) for p in preds])
        order = list(np.flatnonzero(indeg == 0))
        k = 0
        while k < len(order):
            t = order[k]; k += 1
            for u in su[sp[t]:sp[t + 1]]:
                indeg[u] -= 1
                if indeg[u] == 0:
                    order.append(u)
        for t in order:
            m = 0.0
            for p_ in preds[t]:
                if EF[p_] > m:
                    m = EF[p_]; best[t] = p_
            EF[t] = m + d[t]
        end_t = int(np.argmax(EF))
        path = []
        t = end_t
        while t >= 0:
            path.append(t); t = best[t]
        path = path[::-1]
        kinds = {}
        for t in path:
            key = ("diag" if (code[t] // 1000) % 10 == 1 else "off") + ("-last" if code[t] >= 10000 else "-inner")
            kinds[key] = kinds.get(key, 0) + d[t]
        off = 8 + 4 * (nb + 1) + 4 * ns
        ti = np.frombuffer(rest[off:off + 16 * nb], dtype=np.int32).reshape(nb, 4) if len(rest) > off else None
        if ti is not None and slot == 0:
            from collections import Counter
            cnt = Counter()
            for t in path:
                cnt[(int(ti[t, 0]), int(ti[t, 1]), int(ti[t, 2]), int(ti[t, 3]))] += d[t]
            print("  heaviest tiles on the path (I, J, rows I, rows J): us", [(k, round(v, 1)) for k, v in cnt.most_common(6)])
            print("  NT =", int(ti[:, 0].max()) + 1)
        print(f"slot {slot}: critical path {EF[end_t]:.1f} us over {len(path)} tasks (span {span:.1f}); by kind:",
              {k: round(v, 1) for k, v in kinds.items()})
    # queue delay: claim time minus the time the last predecessor finished
    for slot in range(min(S, 1)):
        base_i = slot * nb
        ready = np.zeros(nb)
        for t in range(nb):
            if preds[t]:
                ready[t] = max(end[base_i + p_] for p_ in preds[t])
        qd = claim[base_i:base_i + nb] - ready
        okm = ok[base_i:base_i + nb]
        print(f"queue delay (claim - ready): mean {qd[okm].mean():.1f} us, p50 {np.median(qd[okm]):.1f}, p90 {np.percentile(qd[okm], 90):.1f}, max {qd[okm].max():.1f}")
        # actual path: follow from the last-finishing task the predecessor that finished last
        t = int(np.argmax(end[base_i:base_i + nb] * okm))
        tot_q, tot_d, n = 0.0, 0.0, 0
        while True:
            tot_q += qd[t]; tot_d += dur[base_i + t]; n += 1
            if not preds[t]:
                break
            t = max(preds[t], key=lambda p_: end[base_i + p_])
        print(f"actual last-finisher chain: {n} tasks, task time {tot_d:.1f} us, queue delay {tot_q:.1f} us")
