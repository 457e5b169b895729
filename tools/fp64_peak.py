"""Measure the FP64 GEMM peak of this B200 with cuBLAS (torch.matmul float64),
the denominator of the Jacobian contraction's roofline.
Writes profiles/fp64_peak.json."""
import json, os, sys, time
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(10):
    e0.record(); torch.matmul(a, b, out=c); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n ** 3 / (best / 1e3) / 1e12
t0 = time.time(); k = 0
e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c); k += 1
e1.record(); torch.cuda.synchronize()
sustained = 2 * n ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tflops": burst, "tflops_sustained": sustained, "gpu": torch.cuda.get_device_name(0),
       "how": f"cuBLAS DGEMM via torch.matmul float64 {n}^3: best of 10 (burst) and back to back for 4 s (sustained), CUDA events",
       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
for d in ("profiles", "gpurun_out"):
    os.makedirs(d, exist_ok=True)
    json.dump(out, open(os.path.join(d, "fp64_peak.json"), "w"), indent=1)
print(json.dumps(out))
