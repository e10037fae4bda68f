"""One warmed-up invocation of a hot-path kernel, for ncu targeting
(`ncu -k regex:<kernel> -s <skip> -c <count> python scripts/ncu_target.py <case>`).
Cases: solve32768 (chain solve, C4 1 RHS), solve8192x16 (C3 solve),
batched (C5: 100k x n=32 fused factor + solve), vector (C2: EbV vector path,
n = 1024), update (the n = 32768 step-0 rank-512 trailing update).
Each case runs the call twice (the first warms up); profile the last
launches.  Inputs: the seeded generator (ebv_inputs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ebv_inputs  # noqa: E402
import paper_1907_05767_b200 as ebv  # noqa: E402


def main(case):
    dev = torch.device("cuda:0")
    ctx = ebv.Context(0)
    if case.startswith("solve"):
        n, nrhs = (32768, 1) if case == "solve32768" else (8192, 16)
        d = ebv_inputs.generate(n, seed=1, nrhs=nrhs, device=dev)
        LU, _ = ebv.lu_factor(d["At"].T, ctx=ctx)
        del d["At"]
        for _ in range(2):
            X = ebv.lu_solve(LU, d["B"], ctx=ctx)
        torch.cuda.synchronize()
        print("err", (X - d["X"]).abs().max().item())
    elif case == "batched":
        db = ebv_inputs.generate_batched(100_000, 32, seed=1, nrhs=1, device=dev)
        for _ in range(2):
            At = db["At"].clone()
            Bt = db["B"].transpose(1, 2).contiguous()
            ebv.lu_factor_batched(At, Bt, ctx=ctx)
        torch.cuda.synchronize()
        print("err", (Bt.transpose(1, 2) - db["X"]).abs().max().item())
    elif case == "vector":
        d = ebv_inputs.generate(1024, seed=1, nrhs=1, device=dev)
        ctx.set_path(ebv.EBV_PATH_VECTOR)
        for _ in range(2):
            LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
        torch.cuda.synchronize()
        print("info", int(info))
    elif case == "update":
        n, nb = 32768, 512
        M = n - nb
        A = torch.randn(M, nb, dtype=torch.float64, device=dev).mT.contiguous().mT
        B = torch.randn(nb, M, dtype=torch.float64, device=dev).mT.contiguous().mT
        C = torch.randn(M, M, dtype=torch.float64, device=dev).mT.contiguous().mT
        for _ in range(2):
            ebv.update(C, A, B, ctx=ctx)
        torch.cuda.synchronize()
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main(sys.argv[1])
