"""First-contact GPU probe: GEMM op correctness vs torch (CPU), peaks, filter-step rates."""
import json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D

eng = D.Engine.get(torch.device("cuda", 0))
dev = eng.device
rng = np.random.default_rng(0)
out = {}

def crand(*s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)

# ---- correctness of all op combos, odd sizes
worst = 0.0
for (m, n, k) in [(37, 19, 53), (128, 64, 256), (70, 3, 1000), (5, 7, 4000), (300, 260, 77)]:
    for opa in "NC":
        for opb in "NC":
            A = crand(m, k) if opa == "N" else crand(k, m)
            B = crand(k, n) if opb == "N" else crand(n, k)
            C = crand(m, n)
            al, be = 0.7 - 0.2j, -0.3 + 0.5j
            ref = al * ((A if opa == "N" else A.conj().T) @ (B if opb == "N" else B.conj().T)) + be * C
            dA, dB, dC = D.to_device(A, dev), D.to_device(B, dev), D.to_device(C, dev)
            eng.zgemm(opa, opb, m, n, k, al, dA, dB, be, dC)
            got = D.to_host(dC)
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            worst = max(worst, err)
            if err > 1e-13:
                print("BAD", m, n, k, opa, opb, err)
out["gemm_worst_relerr"] = worst
print("gemm worst", worst, flush=True)

out["peak_dmma_tflops"] = D.peak_dmma_tflops(0, 20000)
out["peak_dfma_tflops"] = D.peak_dfma_tflops(0, 20000)
print("peaks", out["peak_dmma_tflops"], out["peak_dfma_tflops"], flush=True)

# ---- filter step throughput at n=20000
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
g = torch.Generator(device=dev); g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
rates = {}
for k in [1, 16, 26, 32, 64, 128, 210, 275, 512, 1100, 2200]:
    Y1 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    reps = 3 if k >= 512 else 10
    for _ in range(2):
        eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 8.0 * n * n * k / (ms * 1e-3) / 1e12
    rates[k] = (ms, tf)
    print(f"k={k:5d} {ms:9.3f} ms  {tf:6.2f} TFLOP/s", flush=True)
    del Y1, Y0
out["filter_step"] = {str(k): v for k, v in rates.items()}
# cuBLAS zgemm via torch for comparison
for k in [64, 2200]:
    Y = torch.randn((n, k), dtype=torch.complex128, device=dev, generator=g)
    Hm = H.T
    for _ in range(2): torch.matmul(Hm, Y)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): torch.matmul(Hm, Y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out[f"cublas_zgemm_k{k}"] = 8.0 * n * n * k / (ms * 1e-3) / 1e12
    print("cublas k", k, out[f"cublas_zgemm_k{k}"], flush=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
