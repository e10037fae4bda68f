import sys, os
sys.path.insert(0, '/root/repo')
import torch, ebv_inputs, paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0"); ctx = ebv.Context(0)
db = ebv_inputs.generate_batched(100000, 32, seed=1, nrhs=1, device=dev)
LU = db["At"].clone(); ebv.lu_factor_batched(LU, None, ctx=ctx); torch.cuda.synchronize()
B0 = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
ts = []
for r in range(10):
    B = B0.clone(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ebv.lu_solve_batched(LU, B, ctx=ctx); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("solve-only 100k x n=32 x 1 rhs ms", sorted(ts)[5])
