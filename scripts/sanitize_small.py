"""Small invocations of every kernel family (one quick pass over all launch paths;
written for compute-sanitizer, which is closed on this pool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ebv_inputs
import oracle
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
ctx = ebv.Context(0)
for n, nb in ((300, 64), (700, 128), (1537, 64)):
    ctx.set_block(nb)
    d = ebv_inputs.generate(n, seed=n, nrhs=3, device=dev)
    LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
    X = ebv.lu_solve(LU, d["B"], ctx=ctx)
    X2 = ebv.lu_solve(LU, torch.cat([d["B"]] * 30, dim=1), ctx=ctx)   # 90 RHS: TRSM path
    LDU, D = ebv.lu_to_ldu(LU, ctx=ctx)
    An, Bn, sc, inf2 = ebv.normalize_unit_diagonal(d["At"].T, d["B"], ctx=ctx)
torch.cuda.synchronize()
ctx.set_block(0)
ctx.set_path(ebv.EBV_PATH_VECTOR)
d = ebv_inputs.generate(500, seed=2, device=dev)
LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
ctx.set_path(ebv.EBV_PATH_BLOCKED)
for n in (32, 7, 64, 40):
    db = ebv_inputs.generate_batched(50, n, seed=n, nrhs=2, device=dev)
    At = db["At"].clone()
    Bt = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
    ebv.lu_factor_batched(At, Bt, ctx=ctx)
    ebv.lu_solve_batched(At, Bt.clone(), ctx=ctx)
# emulated multi-GPU schedule
n, nb, P = 700, 64, 3
d = ebv_inputs.generate(n, seed=5, nrhs=2, device=dev)
slabs = []
for r in range(P):
    cols = ebv.dist_local_columns(n, nb, r, P, 0)
    slabs.append(d["At"][torch.tensor(cols, dtype=torch.long, device=dev)].clone())
info = torch.zeros((), dtype=torch.int64, device=dev)
sh = torch.cuda.current_stream().cuda_stream
assert ebv.ebv_lu_factor_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n, 0.0,
                                       info.data_ptr(), sh) == 0
B = d["B"].T.clone(memory_format=torch.contiguous_format)
assert ebv.ebv_lu_solve_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n, B.data_ptr(), n,
                                      2, sh) == 0
torch.cuda.synchronize()
print("sanitize workload done")
