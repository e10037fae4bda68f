"""Right- vs left-looking factorization time, and the host-streamed factor
(ebv_lu_factor_host from pinned memory) against copy + factor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
st = torch.cuda.Stream(dev)
info = torch.zeros((), dtype=torch.int64, device=dev)


def timed(fn, reps=3, warm=2):
    ts = []
    for r in range(warm + reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,32768").split(",")]:
    d = ebv_inputs.generate(n, seed=1, device=dev)
    A0 = d["At"]
    Aw = torch.empty_like(A0)
    hA = torch.empty(A0.shape, dtype=torch.float64, pin_memory=True)
    hA.copy_(A0)
    del d
    fl = 2.0 / 3.0 * n ** 3
    for name, path in (("right", ebv.EBV_PATH_BLOCKED), ("left", ebv.EBV_PATH_LEFT)):
        ctx = ebv.Context(0, path=path)
        ctx.set_graphs(False)

        def run():
            with torch.cuda.stream(st):
                Aw.copy_(A0)
            ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), st.cuda_stream)
        ms = timed(run)
        print(json.dumps({"n": n, "schedule": name, "what": "device copy + factor", "ms": ms,
                          "tflops": fl / ms / 1e9}), flush=True)

        def run_h2d():
            with torch.cuda.stream(st):
                Aw.copy_(hA, non_blocking=True)
            ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), st.cuda_stream)
        ms = timed(run_h2d)
        print(json.dumps({"n": n, "schedule": name, "what": "H2D copy then factor", "ms": ms,
                          "tflops": fl / ms / 1e9}), flush=True)
    ctx = ebv.Context(0)

    def run_host():
        ebv.ebv_lu_factor_host(ctx.handle, n, hA.data_ptr(), n, Aw.data_ptr(), n, 0.0, info.data_ptr(),
                               st.cuda_stream)
    ms = timed(run_host)
    assert int(info) == 0
    print(json.dumps({"n": n, "schedule": "default host path", "what": "ebv_lu_factor_host (pinned)", "ms": ms,
                      "tflops": fl / ms / 1e9}), flush=True)
    del A0, Aw, hA
