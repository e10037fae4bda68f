"""Does a concurrent host->device copy slow the factorization (the e2e gap)?
Factor n = 32768 alone, then with the next step's 8.6 GB H2D copy from
pinned memory running on another stream, then with that copy split into
chunks (same bytes, lower peak rate).  python scripts/h2d_interference.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

n = int(os.environ.get("N", "32768"))
dev = torch.device("cuda:0")
A0 = ebv_inputs.generate(n, seed=1, device=dev, with_b=False)["At"]
A = torch.empty_like(A0)
A2 = torch.empty_like(A0)
hA = torch.empty(A0.shape, dtype=torch.float64, pin_memory=True)
hA.copy_(A0)
info = torch.zeros((), dtype=torch.int64, device=dev)
ctx = ebv.Context(0)
s = torch.cuda.Stream(dev)
cs = torch.cuda.Stream(dev)


def factor_ms(copy_mode):
    A.copy_(A0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    cs.wait_event(e0)
    with torch.cuda.stream(cs):
        c0.record(cs)
        if copy_mode == "whole":
            A2.copy_(hA, non_blocking=True)
        elif copy_mode == "rows":   # the same bytes as 64 column-slab copies
            step = n // 64
            for j in range(0, n, step):
                A2[j:j + step].copy_(hA[j:j + step], non_blocking=True)
        c1.record(cs)
    ebv.ebv_lu_factor(ctx.handle, n, A.data_ptr(), n, 0.0, info.data_ptr(), s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (c0.elapsed_time(c1) if copy_mode else 0.0)


for rep in range(2):
    for mode in (None, "whole", None, "rows"):
        t, tc = factor_ms(mode)
        print(json.dumps({"n": n, "copy": mode, "factor_ms": round(t, 2), "copy_ms": round(tc, 1)}), flush=True)
