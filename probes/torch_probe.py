"""Probe M1/M5: cuBLAS float64 GEMM throughput (burst and
sustained, with clocks) and fp64 device copy bandwidth.  Context numbers only:
cuBLAS is a comparator, never on the product path."""
import json
import subprocess
import time

import torch


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                              "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception as e:  # noqa: BLE001
        return str(e)


def main():
    dev = torch.device("cuda:0")
    for n in (4096, 8192, 16384):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(2):
            c = a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"probe": "M1_dgemm_burst", "n": n, "ms": best, "tflops": 2 * n ** 3 / best / 1e9}))
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t0 = time.time(); cnt = 0
    e0.record()
    while time.time() - t0 < 4.0:
        c = a @ b; cnt += 1
        if cnt % 10 == 0:
            torch.cuda.synchronize()
            clk = clocks()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"probe": "M1_dgemm_sustained", "n": n, "count": cnt, "tflops": 2 * n ** 3 * cnt / ms / 1e9, "clocks": clk}))
    # M5: fp64 copy bandwidth
    x = torch.empty(2 ** 28, dtype=torch.float64, device=dev).fill_(1.0)
    y = torch.empty_like(x)
    for _ in range(3):
        y.copy_(x)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"probe": "M5_copy", "bytes": 2 * x.numel() * 8, "gbs": 2 * x.numel() * 8 / best / 1e6}))
    # cuSOLVER no-pivot LU comparator at n=8192 (context only)
    try:
        n = 8192
        A = torch.rand(n, n, dtype=torch.float64, device=dev) * 2 - 1
        A += torch.diag(A.abs().sum(1) + 1)
        for _ in range(2):
            LU, piv = torch.linalg.lu_factor(A, pivot=False)
        torch.cuda.synchronize()
        e0.record(); LU, piv = torch.linalg.lu_factor(A, pivot=False); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"probe": "cusolver_getrf_nopivot", "n": n, "ms": ms, "gflops": 2 / 3 * n ** 3 / ms / 1e6}))
        e0.record(); LU, piv = torch.linalg.lu_factor(A, pivot=True); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"probe": "cusolver_getrf_pivot", "n": n, "ms": ms, "gflops": 2 / 3 * n ** 3 / ms / 1e6}))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"probe": "cusolver", "error": str(e)}))


if __name__ == "__main__":
    main()
