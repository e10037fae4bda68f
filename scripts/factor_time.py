"""Median time of ebv_lu_factor (default schedule, CUDA-graph replay) at the
given orders: python scripts/factor_time.py 8192 16384 [--reps 5]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int, nargs="+")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--graphs", type=int, default=1, help="CUDA-graph replay of the schedule (ebv_set_graphs)")
ap.add_argument("--stats", type=int, default=0, help="library per-launch statistics on (disables graphs)")
ap.add_argument("--legacy", action="store_true", help="the legacy default stream instead of a created one")
ap.add_argument("--nb", type=int, default=0, help="block width (0: size-adaptive)")
ap.add_argument("--leaf", type=int, default=0, help="leaf width (0: 64)")
a = ap.parse_args()
dev = torch.device("cuda:0")
ctx = ebv.Context(0)
ctx.set_graphs(bool(a.graphs))
ctx.set_leaf(a.leaf)
ctx.set_block(a.nb)
ctx.stats_enable(bool(a.stats))
s = torch.cuda.default_stream(dev) if a.legacy else torch.cuda.Stream(dev)
for n in a.n:
    A0 = ebv_inputs.generate(n, seed=1, device=dev, with_b=False)["At"]
    A = A0.clone()
    info = torch.zeros((), dtype=torch.int64, device=dev)
    ts = []
    with torch.cuda.stream(s):
        for r in range(a.reps + 3):
            A.copy_(A0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ebv.ebv_lu_factor(ctx.handle, n, A.data_ptr(), n, 0.0, info.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            if r >= 3:
                ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"n": n, "ms_median": ts[len(ts) // 2], "ms_min": ts[0], "u12la": os.environ.get("EBV_U12_LA", "auto"), "graphs": a.graphs, "nb": ctx.block_width(n), "leaf": a.leaf or 64, "stats": a.stats, "legacy": a.legacy,
                      "tflops": 2 / 3 * n ** 3 / (ts[len(ts) // 2] * 1e-3) / 1e12}), flush=True)
    del A, A0
