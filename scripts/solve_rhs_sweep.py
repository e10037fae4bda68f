"""ebv_lu_solve time vs number of right-hand sides (run twice: EBV_SOLVE_TRSM_RHS=1 forces the
TRSM path, a huge value forces the wavefront kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
s = torch.cuda.Stream(dev)
ctx = ebv.Context(0)
for n in (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4096,8192").split(",")):
    d = ebv_inputs.generate(n, seed=1, device=dev)
    with torch.cuda.stream(s):
        LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
        for nr in (1, 2, 4, 16, 32, 64, 65, 128, 256, 1024):
            B0 = torch.randn(nr, n, dtype=torch.float64, device=dev)
            Bw = torch.empty_like(B0)
            ts = []
            for rep in range(5):
                Bw.copy_(B0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                st = ebv.ebv_lu_solve(ctx.handle, n, LU.data_ptr(), n,
                                      Bw.data_ptr(), n, nr, s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                assert st == 0
                if rep >= 2:
                    ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            print(json.dumps({"n": n, "nrhs": nr, "ms": ms, "gflops": 2.0 * n * n * nr / ms / 1e6,
                              "path_env": os.environ.get("EBV_SOLVE_TRSM_RHS", "default")}), flush=True)
