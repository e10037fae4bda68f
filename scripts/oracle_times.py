"""The serial CPU oracle (oracle/, test infrastructure) timed on the host's
cores at the BASELINE.json configs: C1 (n = 64, median of 200), C2 (n = 1024,
median of 3), C5 (100k x n = 32 systems, one run), and n = 4096 (one run),
from which C3 / C4 are extrapolated as t(4096) * (n / 4096)^3 (labelled).
One thread (the oracle is serial).  JSON lines."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import ebv_inputs  # noqa: E402
import oracle  # noqa: E402


def t_solve(n, reps):
    d = ebv_inputs.generate(n, seed=1, nrhs=1)
    a, b = d["At"].T.numpy().copy(), d["B"].numpy().copy()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        lu, info = oracle.lu_factor(a)
        x = oracle.lu_solve(lu, b)
        ts.append(time.perf_counter() - t0)
    assert info == 0 and np.max(np.abs(x - d["X"].numpy())) <= 1e-10
    return statistics.median(ts)


def main():
    oracle.build()
    cpu = open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ") if os.path.exists("/proc/cpuinfo") else "?"
    head = {"cpu": cpu, "nproc": os.cpu_count(), "threads_used": 1}
    for cfg, n, reps in (("C1", 64, 200), ("C2", 1024, 3), ("n4096", 4096, 1)):
        t = t_solve(n, reps)
        print(json.dumps({**head, "config": cfg, "n": n, "oracle_factor_solve_ms": 1e3 * t,
                          "gflops": 2 / 3 * n ** 3 / t / 1e9}), flush=True)
        if cfg == "n4096":
            for c2, n2 in (("C3", 8192), ("C4", 32768)):
                print(json.dumps({**head, "config": c2, "n": n2, "oracle_factor_solve_ms_extrapolated":
                                  1e3 * t * (n2 / 4096) ** 3, "note": "t(4096) * (n/4096)^3, not measured"}), flush=True)
    db = ebv_inputs.generate_batched(100_000, 32, seed=1, nrhs=1)
    a, b = db["At"].transpose(1, 2).numpy().copy(), db["B"].numpy().copy()
    t0 = time.perf_counter()
    lu, x, info = oracle.lu_factor_batched(a, b)
    t = time.perf_counter() - t0
    assert not info.any()
    print(json.dumps({**head, "config": "C5", "batch": 100000, "n": 32, "oracle_factor_solve_ms": 1e3 * t}), flush=True)


if __name__ == "__main__":
    main()
