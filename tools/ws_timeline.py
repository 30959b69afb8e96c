"""Per-SM consumer timeline of one warp-specialised factor launch (PINLA_TRACE dump):
where the MMA team's time goes -- pair loop vs finalize vs stores vs publish vs the gap to the
next task on the same SM -- and the pair loop's rate against the DMMA peak.

    PINLA_TRACE=gpurun_out/tr.bin python tools/prof_case.py c4 '{"nt": 16, "m": 128000}' 3 1
    python tools/ws_timeline.py gpurun_out/tr.bin
"""
import sys
import numpy as np

f = open(sys.argv[1], "rb")
nb, S = np.frombuffer(f.read(16), dtype=np.int64)
tk = np.frombuffer(f.read(16 * nb), dtype=np.int32).reshape(nb, 4)
tr = np.frombuffer(f.read(8 * 8 * nb * S), dtype=np.uint64).reshape(nb * S, 8).astype(np.float64)
code = np.frombuffer(f.read(8 * nb), dtype=np.int64)
ok = (tr[:, 2] > 0) & (tr[:, 5] > 0)
base = np.arange(nb * S) % nb
pairs = (code[base] % 1000).astype(np.float64)
diag = (code[base] // 1000) % 10 == 1
last = code[base] >= 10000
t0 = tr[ok, 4].min()
us = lambda c: (tr[:, c] - t0) / 1e3
ready, pend, done, smid, pop, cbeg, fin, sto = us(0), us(1), us(2), tr[:, 3], us(4), us(5), us(6), us(7)
span = done[ok].max()
print(f"tasks {ok.sum()} slots {S} span {span:.1f} us")
tot = dict(pairs=0.0, finalize=0.0, stores=0.0, publish=0.0, gap=0.0, head=0.0)
nsm = 0
for sm in np.unique(smid[ok]):
    idx = np.flatnonzero(ok & (smid == sm))
    idx = idx[np.argsort(cbeg[idx])]
    nsm += 1
    tot["pairs"] += (pend[idx] - cbeg[idx]).sum()
    lf = idx[last[idx]]
    tot["finalize"] += (fin[lf] - pend[lf]).sum()
    tot["stores"] += (sto[lf] - fin[lf]).sum()
    tot["publish"] += (done[lf] - sto[lf]).sum()
    nl = idx[~last[idx]]
    tot["publish"] += (done[nl] - pend[nl]).sum()  # store + publish of inner chunks
    tot["gap"] += (cbeg[idx][1:] - done[idx][:-1]).sum()
    tot["head"] += cbeg[idx][0] + (span - done[idx][-1])
wall = nsm * span
print(f"SMs {nsm}; consumer time shares of {wall/1e3:.1f} SM-ms:")
for k, v in tot.items():
    print(f"  {k:9s} {v/1e3:9.2f} ms  {100*v/wall:5.1f} %")
m = ok & (pairs > 0)
per_pair = (pend[m] - cbeg[m]).sum() / pairs[m].sum()
print(f"pair loop: {per_pair:.3f} us per 64x64x64 pair = {2*64**3/per_pair/1e6*nsm:.2f} TF/s-equivalent over {nsm} SMs")
for name, mm in (("last-off", last & ~diag), ("last-diag", last & diag), ("inner", ~last)):
    mm = mm & ok
    if mm.sum():
        print(f"  {name:9s} n={mm.sum():7d} mean pairs {pairs[mm].mean():5.2f} pair-loop {np.mean(pend[mm]-cbeg[mm]):6.2f} us "
              f"tail {np.mean(done[mm]-pend[mm]):6.2f} us; ready->begin {np.median(cbeg[mm]-ready[mm]):6.2f} us (median)")
inner = ok & ~last & (code[base] < 1000)
tail = done - pend
print(f"inner chunk tasks continued on the same SM (tail < 0.5 us: no store / publish): "
      f"{(tail[inner] < 0.5).sum()} of {inner.sum()} ({100*(tail[inner] < 0.5).mean():.1f} %)")
if len(sys.argv) > 2 and sys.argv[2] == "ringwait":
    # diagnostic build (-DPINLA_WS_TRACE_WAIT): trace word 6 of an inner task = SM clocks thread 0 waited for ring stages
    rw = tr[:, 6][inner] / 1.965e3  # us at 1965 MHz
    pl = (pend - cbeg)[inner]
    print(f"inner tasks: ring-stage wait {rw.sum()/1e3:.1f} ms of {pl.sum()/1e3:.1f} ms pair-loop time "
          f"({100*rw.sum()/pl.sum():.1f} %); per task mean {rw.mean():.2f} us, p90 {np.percentile(rw, 90):.2f} us")
