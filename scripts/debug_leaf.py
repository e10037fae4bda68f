"""Locate the first entry where the blocked factorization differs from the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ebv_inputs
import oracle
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
for n, nb, la in ((1537, 64, 1), (1537, 64, 0), (300, 64, 1), (130, 64, 1), (65, 64, 1), (64, 64, 1), (200, 128, 1)):
    d = ebv_inputs.generate(n, seed=5, device=dev)
    ctx = ebv.Context(0)
    ctx.set_block(nb)
    ctx.set_lookahead(bool(la))
    LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
    torch.cuda.synchronize()
    g = LU.cpu().numpy()
    o, _ = oracle.lu_factor(d["At"].T.cpu().numpy())
    diff = np.argwhere(g.view(np.uint64) != o.view(np.uint64))
    print(n, nb, la, "ndiff", len(diff), "first", diff[:5].tolist(), flush=True)
    if len(diff):
        i, j = diff[0]
        print("   g", g[i, j], "o", o[i, j], "rel", abs(g[i, j] - o[i, j]) / abs(o[i, j]))
