"""Lower bound of the blocked schedule at n (default 8192): the sum of its
trailing-update DMMA launches timed standalone (no panel work)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.randn(n, n, dtype=torch.float64, device=dev)   # storage; column-major views below
ctx = ebv.Context(0)
s = torch.cuda.current_stream(dev).cuda_stream
for nb in (128, 256):
    tot = 0.0
    for c0 in range(0, n - nb, nb):
        rest = n - c0 - nb
        M = N = rest
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        base = A.data_ptr()
        # L21 at rows c0+nb.., cols c0..; U12 rows c0.., cols c0+nb..; C at (c0+nb, c0+nb)
        Lp = base + 8 * ((c0 + nb) + c0 * n)
        Up = base + 8 * (c0 + (c0 + nb) * n)
        Cp = base + 8 * ((c0 + nb) + (c0 + nb) * n)
        ebv.ebv_update(ctx.handle, M, N, nb, Lp, n, Up, n, Cp, n, s)
        e0.record()
        ebv.ebv_update(ctx.handle, M, N, nb, Lp, n, Up, n, Cp, n, s)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    fl = 2.0 / 3.0 * n ** 3
    print(json.dumps({"n": n, "nb": nb, "trailing_updates_ms": tot, "tflops_if_only_these": fl / tot / 1e9}), flush=True)
