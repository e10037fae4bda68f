"""The README usage example at small sizes (dense, batched medium, band storage): python scripts/readme_example.py"""
import sys
sys.path.insert(0, "/root/repo")
import torch, ebv_inputs
import paper_1907_05767_b200 as ebv
ctx = ebv.Context(0)
d = ebv_inputs.generate(1024, seed=1, nrhs=16, device="cuda")
A, B = d["At"].T, d["B"]
LU, info = ebv.lu_factor(A, ctx=ctx)
X = ebv.lu_solve(LU, B, ctx=ctx)
print("dense", int(info), (X - d["X"]).abs().max().item())
db = ebv_inputs.generate_batched(100, 200, seed=1, nrhs=2, device="cuda")
At = db["At"].clone(); Bt = db["B"].transpose(1, 2).contiguous()
info = ebv.lu_factor_batched(At, Bt, ctx=ctx)
print("batched", int(info.abs().sum()), (Bt.transpose(1, 2) - db["X"]).abs().max().item())
g = ebv_inputs.generate_band(1 << 16, 64, 64, ebv.EBV_BAND_PAD, ebv.band_ld(64, 64), device="cuda")
AB, info = ebv.lu_factor_band(g["AB"], 1 << 16, 64, 64, ctx=ctx)
x = ebv.lu_solve_band(AB, g["B"], 64, 64, ctx=ctx)
print("band", int(info), (x - g["X"]).abs().max().item())
