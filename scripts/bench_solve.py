"""Time ebv_lu_solve (Eq 1) at the configs' orders: CUDA events on the
launching stream, warm-up, median of reps; prints one JSON line per case.
EBV_SOLVE_CHAIN=0 in the environment selects the wavefront kernel."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ebv_inputs  # noqa: E402
import paper_1907_05767_b200 as ebv  # noqa: E402


def main():
    cases = [(1024, 1), (8192, 1), (8192, 16), (32768, 1), (32768, 4), (16384, 1)]
    if len(sys.argv) > 1:
        cases = [tuple(int(x) for x in c.split("x")) for c in sys.argv[1:]]
    dev = torch.device("cuda:0")
    ctx = ebv.Context(0)
    s = torch.cuda.Stream(dev)
    torch.cuda.set_stream(s)
    for n, nrhs in cases:
        d = ebv_inputs.generate(n, seed=1, nrhs=nrhs, device=dev)
        LU, _ = ebv.lu_factor(d["At"].T, ctx=ctx)
        del d["At"]
        B0 = ebv.colmajor_copy(d["B"])
        X = B0.clone()
        ts = []
        for r in range(8):
            X.copy_(B0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ebv.lu_solve(LU, X, ctx=ctx, inplace=True)
            e1.record(s)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        err = (X - d["X"]).abs().max().item()
        ms = statistics.median(ts)
        by = 8.0 * n * n + 32.0 * n * nrhs
        print(json.dumps({"n": n, "nrhs": nrhs, "ms": ms, "min_ms": min(ts), "max_ms": max(ts),
                          "gbs": by / ms / 1e6, "frac_hbm": by / ms / 1e6 / 6545.6, "err": err,
                          "kernel": "wavefront" if os.environ.get("EBV_SOLVE_CHAIN") == "0" else "chain"}),
              flush=True)
        del LU, X, B0, d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
