import sys, os
sys.path.insert(0, '/root/repo')
import torch, ebv_inputs, paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
ctx = ebv.Context(0)
for n in (48, 64, 40, 33):
    for nrhs in (0, 1, 2):
        db = ebv_inputs.generate_batched(100000, n, seed=1, nrhs=max(nrhs,1), device=dev)
        A0 = db["At"]; B0 = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)[:, :nrhs].contiguous() if nrhs else None
        ts = []
        for r in range(6):
            A = A0.clone(); B = B0.clone() if nrhs else None
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ebv.lu_factor_batched(A, B, ctx=ctx)
            e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(n, nrhs, sorted(ts)[2])
