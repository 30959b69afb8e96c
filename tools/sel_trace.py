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
