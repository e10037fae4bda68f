"""Median time of the EbV vector path (EBV_PATH_VECTOR) and the blocked path
at n (default 1024): CUDA events on a created stream, warm-up 3, median of 9."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ebv_inputs  # noqa: E402
import paper_1907_05767_b200 as ebv  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = torch.device("cuda:0")
s = torch.cuda.Stream(dev)
torch.cuda.set_stream(s)
ctx = ebv.Context(0)
A0 = ebv_inputs.generate(n, seed=1, device=dev)["At"]
A = A0.clone()
info = torch.zeros((), dtype=torch.int64, device=dev)
for path, name in ((ebv.EBV_PATH_VECTOR, "vector"), (ebv.EBV_PATH_BLOCKED, "blocked")):
    ctx.set_path(path)
    ts = []
    for r in range(12):
        A.copy_(A0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ebv.ebv_lu_factor(ctx.handle, n, A.data_ptr(), n, 0.0, info.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    print(name, n, "%.3f ms" % statistics.median(ts))
