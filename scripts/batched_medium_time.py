"""Batched medium orders (the blocked schedule over the whole batch):
factor + 1-RHS solve times.  python scripts/batched_medium_time.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
ctx = ebv.Context(0)
for batch, n in ((20000, 128), (4000, 256), (800, 512)):
    db = ebv_inputs.generate_batched(batch, n, seed=1, nrhs=1, device=dev)
    A0 = db["At"]
    B0 = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
    ts = []
    for r in range(6):
        A, B = A0.clone(), B0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ebv.lu_factor_batched(A, B, ctx=ctx)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(batch, n, "ms", round(sorted(ts)[3], 3))
    del db, A0, B0
