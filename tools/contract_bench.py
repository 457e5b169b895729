"""Time the DMMA Jacobian contraction alone at the bench shape (values only)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05586_b200 as dot
nb, ld, ls, K, n_p = 3, 256, 256, 4012, 80
g = torch.Generator(device="cuda").manual_seed(0)
Lam = torch.randn(nb, ld, K, dtype=torch.complex128, device="cuda", generator=g)
U = torch.randn(nb, ls, K, dtype=torch.complex128, device="cuda", generator=g)
G = torch.randn(K, n_p, dtype=torch.float64, device="cuda", generator=g)
for _ in range(3):
    J = dot.contract(Lam, U, G)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(10):
    e0.record(); J = dot.contract(Lam, U, G); e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
t = min(ms)
fl = 4.0 * nb * ld * ls * K * n_p
# spot check against torch (complex Hadamard then real GEMM), one frequency, a few pairs
b = 1
H = (Lam[b][:, None, :] * U[b][None, :4, :]).reshape(-1, K)
ref = -(H @ G.to(torch.complex128))
err = (J[b][:, :4, :].reshape(-1, n_p) - ref).abs().max().item() / ref.abs().max().item()
print(json.dumps({"ms": t, "tflops": fl / t / 1e9, "rel_err_vs_torch": err}))
