"""Measure the fp64 GEMM roofline denominator on a B200: cuBLAS DGEMM via torch.

Burst = best of 10 single 8192^3 DGEMMs; sustained = back-to-back for ~4 s.
Writes gpurun_out/fp64_peak.json (copied into profiles/ by hand).
"""
import json, time, torch

def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n**3 / (best * 1e-3) / 1e12
    t0 = time.time(); k = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c); k += 1
        if k % 8 == 0: torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sust = 2 * n**3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
    out = {"fp64_dgemm_tflops": burst, "fp64_dgemm_tflops_sustained": sust, "n": n,
           "how": "torch.matmul fp64 (cuBLAS DGEMM) 8192^3, best of 10 / back-to-back 4 s"}
    print(json.dumps(out))
    json.dump(out, open("gpurun_out/fp64_peak.json", "w"), indent=1)

if __name__ == "__main__":
    main()
