"""One blocked factorization (after a warm-up) for launch-list / ncu profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda:0")
d = ebv_inputs.generate(a.n, seed=1, device=dev)
A0 = d["At"]
ctx = ebv.Context(0)
for r in range(a.reps):
    A = A0.clone()
    LU, info = ebv.lu_factor(A.T, ctx=ctx, inplace=True)
    torch.cuda.synchronize()
print("info", int(info), "launches", ctx.launch_count())
