"""Correctness of the DMMA update C -= A B against torch (cuBLAS) at many shapes,
and n=4096 factor vs oracle (leading block)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1907_05767_b200 as ebv
import ebv_inputs, oracle

dev = torch.device("cuda:0")
torch.manual_seed(0)
def cm(r, c):
    return torch.randn(c, r, dtype=torch.float64, device=dev).T
bad = 0
for M, N, K in [(128, 64, 16), (256, 128, 256), (1000, 999, 77), (3840, 3840, 256), (4096, 4096, 256), (3840, 64, 64),
                (64, 3840, 64), (128, 3840, 128), (8192, 8192, 256), (5000, 300, 600), (300, 5000, 600), (4096, 4096, 4096)]:
    C, A, B = cm(M, N), cm(M, K), cm(K, N)
    ref = C - A @ B
    ebv.update(C, A, B)
    torch.cuda.synchronize()
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    # locate bad tiles
    msg = ""
    if err > 1e-13:
        bad += 1
        badm = ((C - ref).abs() > 1e-10 * ref.abs().max())
        idx = badm.nonzero()
        msg = f" nbad={idx.shape[0]} first={idx[:5].tolist()} rows[{idx[:,0].min().item()},{idx[:,0].max().item()}] cols[{idx[:,1].min().item()},{idx[:,1].max().item()}]"
    print(f"M={M} N={N} K={K} relerr={err:.3e}{msg}", flush=True)
n = int(os.environ.get("CHECK_N", "4096"))
d = ebv_inputs.generate(n, seed=9, device=dev)
A = d["At"].T
LU, info = ebv.lu_factor(A)
torch.cuda.synchronize()
m = 1024
lu_o, _ = oracle.lu_factor(A[:m, :m].cpu().numpy())
print("factor n", n, "leading", m, "bitwise", np.array_equal(LU[:m, :m].cpu().numpy(), lu_o), "tma env", os.environ.get("EBV_GEMM_TMA"))
L = torch.tril(LU, -1) + torch.eye(n, device=dev, dtype=torch.float64)
U = torch.triu(LU)
rec = (L @ U - A).abs()
print("reconstruction max", rec.max().item())
bi = (rec > 1e-10).nonzero()
if bi.shape[0]:
    print("bad entries", bi.shape[0], "rows", bi[:,0].min().item(), bi[:,0].max().item(), "cols", bi[:,1].min().item(), bi[:,1].max().item(), bi[:8].tolist())
print("bad gemm shapes", bad)
