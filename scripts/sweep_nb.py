"""Factor time vs block width nb (and lookahead on/off) at the given sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)   # non-default: CUDA Graph replay applies
ctx = ebv.Context(0)
info = torch.zeros((), dtype=torch.int64, device=dev)
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,32768").split(",")]:
    d = ebv_inputs.generate(n, seed=1, device=dev)
    A0 = d["At"]
    Aw = torch.empty_like(A0)
    del d
    nbs = ((0, 1), (128, 1), (256, 1), (512, 1), (-1, 0))
    if len(sys.argv) >= 3:
        nbs = tuple((int(x), 1) for x in sys.argv[2].split(","))
    for nb, la in nbs:
        ctx.set_block(nb)
        ctx.set_lookahead(bool(la))
        ts = []
        for r in range(4):
            with torch.cuda.stream(stream):
                Aw.copy_(A0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts[2:])
        print(json.dumps({"n": n, "nb": nb, "lookahead": la, "ms": ms, "tflops": 2 / 3 * n ** 3 / ms / 1e9}), flush=True)
    ctx.set_block(0)
    ctx.set_lookahead(True)
    ctx.set_graphs(False)
    with torch.cuda.stream(stream):
        Aw.copy_(A0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    print(json.dumps({"n": n, "nb": 0, "graphs": 0, "ms": e0.elapsed_time(e1)}), flush=True)
    ctx.set_graphs(True)
    del A0, Aw
