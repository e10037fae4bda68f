"""Where the DMMA update loses against its isolated rate inside the
factorization: class statistics (per-launch events, graphs off) with the
lookahead on and off.  python scripts/update_insitu.py [--n 32768]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
a = ap.parse_args()
dev = torch.device("cuda:0")
n = a.n
A0 = ebv_inputs.generate(n, seed=1, device=dev, with_b=False)["At"]
A = torch.empty_like(A0)
info = torch.zeros((), dtype=torch.int64, device=dev)
s = torch.cuda.Stream(dev)
for la in (True, False):
    ctx = ebv.Context(0)
    ctx.set_lookahead(la)
    with torch.cuda.stream(s):
        for rep in range(2):
            A.copy_(A0)
            torch.cuda.synchronize()
            if rep == 1:
                ctx.stats_reset()
                ctx.stats_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ebv.ebv_lu_factor(ctx.handle, n, A.data_ptr(), n, 0.0, info.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
    st = ctx.stats()
    ctx.stats_enable(False)
    out = {"n": n, "lookahead": la, "factor_ms": e0.elapsed_time(e1)}
    for k, v in st.items():
        if v["launches"]:
            out[k] = {"launches": v["launches"], "ms": round(v["ms"], 3),
                      "tflops": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] > 0 else None}
    print(json.dumps(out), flush=True)
    del ctx
