"""Vector-path factorization (for ncu of vector_lu_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--ctas", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda:0")
ctx = ebv.Context(0)
ctx.set_path(ebv.EBV_PATH_VECTOR)
ctx.set_vector_ctas(a.ctas)
d = ebv_inputs.generate(a.n, seed=1, device=dev)
for _ in range(2):
    LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
torch.cuda.synchronize()
print("ok", int(info))
