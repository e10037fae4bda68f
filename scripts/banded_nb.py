"""Banded (stencil) factor time vs block width."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
st = torch.cuda.Stream(dev)
info = torch.zeros((), dtype=torch.int64, device=dev)
for m in (128, 256):
    n = m * m
    A0 = ebv_inputs.generate(n, seed=1, device=dev, stencil_m=m, with_b=False)["At"]
    Aw = torch.empty_like(A0)
    for nb in (64, 128, 256, 512):
        ctx = ebv.Context(0)
        ctx.set_block(nb)
        ts = []
        for r in range(4):
            with torch.cuda.stream(st):
                Aw.copy_(A0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            ebv.ebv_lu_factor_banded(ctx.handle, n, m, m, Aw.data_ptr(), n, 0.0, info.data_ptr(), st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(json.dumps({"n": n, "m": m, "nb": nb, "ms": min(ts[1:])}), flush=True)
    del A0, Aw
