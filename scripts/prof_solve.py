"""One factor + solve (for ncu of the solve / batched kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--nrhs", type=int, default=16)
ap.add_argument("--batched", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda:0")
if a.batched:
    db = ebv_inputs.generate_batched(a.batched, 32, seed=1, nrhs=1, device=dev)
    At = db["At"].clone(); Bt = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
    for _ in range(2):
        ebv.lu_factor_batched(At.clone(), Bt.clone())
    torch.cuda.synchronize()
else:
    d = ebv_inputs.generate(a.n, seed=1, nrhs=a.nrhs, device=dev)
    LU, info = ebv.lu_factor(d["At"].T)
    for _ in range(2):
        X = ebv.lu_solve(LU, d["B"])
    torch.cuda.synchronize()
print("ok")
