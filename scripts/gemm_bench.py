"""DMMA update (C -= A B) throughput at the shapes the factorizations use."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
ctx = ebv.Context(0)
def cm(r, c):
    return torch.randn(c, r, dtype=torch.float64, device=dev).T
shapes = [tuple(int(v) for v in x.split("x")) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [(16384, 16384, 16384), (8192, 8192, 8192), (4096, 4096, 4096), (32512, 32512, 256),
          (16384, 16384, 256), (8064, 8064, 128), (8192, 8192, 64), (16384, 64, 64), (64, 16384, 64),
          (4096, 4096, 64), (2048, 2048, 2048), (1024, 1024, 1024)]
print(json.dumps({"variant_env": os.environ.get("EBV_GEMM_TMA", "0")}), flush=True)
for M, N, K in shapes:
    C, A, B = cm(M, N), cm(M, K), cm(K, N)
    ebv.update(C, A, B, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        ebv.update(C, A, B, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"M": M, "N": N, "K": K, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9,
                      "gbs_C": 16 * M * N / ms / 1e6}), flush=True)
    del C, A, B
