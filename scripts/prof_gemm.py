"""One DMMA update C -= A B of a given shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
import paper_1907_05767_b200 as ebv
ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=8192)
ap.add_argument("--N", type=int, default=8192)
ap.add_argument("--K", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dev = torch.device("cuda:0")
def cm(r, c):
    return torch.randn(c, r, dtype=torch.float64, device=dev).T
C, A, B = cm(a.M, a.N), cm(a.M, a.K), cm(a.K, a.N)
for _ in range(a.reps):
    ebv.update(C, A, B)
torch.cuda.synchronize()
print("ok")
