"""Summaries of ncu output for profiles/ (run here, on the files gpurun
brought back).

    python tools/ncu_summary.py full  gpurun_out/factor_TAG.ncu-rep  [out.json]
    python tools/ncu_summary.py shares gpurun_out/launches_TAG.csv   [out.csv]

`full`: one --set full capture -> duration, DRAM traffic, DMMA / fp64 pipe
utilisation, occupancy, top warp stalls (pc sampling).
`shares`: a --metrics gpu__time_duration.sum launch list -> per-kernel launch
count, total time and share (cold-cache serialised times: compare SHARES).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    return [{name: (unit, val) for name, unit, val in zip(h, u, row)} for row in r[2:]]


def num(d, key, scale=1.0):
    if key not in d:
        return None
    unit, val = d[key]
    try:
        x = float(val.replace(",", ""))
    except ValueError:
        return None
    mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
            "ns": 1e-9, "s": 1.0}.get(unit, 1.0)
    return x * mult * scale


def full(rep, out):
    res = []
    for d in raw_rows(rep):
        stalls = {}
        for k, (unit, val) in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(val.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = dict(sorted(((k, round(100 * v / tot, 1)) for k, v in stalls.items()),
                          key=lambda kv: -kv[1])[:8])
        rd = num(d, "dram__bytes_read.sum")
        wr = num(d, "dram__bytes_write.sum")
        res.append({
            "kernel": d.get("Kernel Name", ("", ""))[1].split("(")[0],
            "grid": d.get("Grid Size", ("", ""))[1], "block": d.get("Block Size", ("", ""))[1],
            "gpu_time_s": num(d, "gpu__time_duration.sum"),
            "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_launch": (rd or 0) + (wr or 0),
            "dram_throughput_pct": num(d, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dmma_inst_pct_of_peak_active": num(d, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
            "tensor_pipe_active_pct_elapsed": num(d, "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_active_pct": num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": num(d, "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers_per_thread": num(d, "launch__registers_per_thread"),
            "top_stalls_pct": top,
        })
    js = json.dumps(res if len(res) > 1 else res[0], indent=1)
    if out:
        open(out, "w").write(js + "\n")
    print(js)


def shares(path, out):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    for row in csv.DictReader(lines[start:]):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = row["Kernel Name"].split("(")[0].split("<")[0].strip()
        if k.startswith("void "):
            k = k[5:]
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(row["Metric Unit"], 1.0)
        tot[k] += float(row["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    s = sum(tot.values())
    rows = sorted(tot, key=lambda k: -tot[k])
    text = "kernel,launches,total_us,share\n" + "".join(
        f"{k},{cnt[k]},{tot[k]:.1f},{tot[k] / s:.3f}\n" for k in rows)
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    {"full": full, "shares": shares}[mode](path, out)
