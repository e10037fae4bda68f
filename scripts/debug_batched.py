"""Debug: batched kernel vs oracle, print first mismatches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ebv_inputs, oracle
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
for n, batch, nrhs in [(32, 4, 1), (32, 1, 1), (5, 2, 1)]:
    db = ebv_inputs.generate_batched(batch, n, seed=7, nrhs=nrhs, device=dev)
    At = db["At"].clone()
    Bt = db["B"].transpose(1, 2).contiguous()
    info = ebv.lu_factor_batched(At, Bt)
    torch.cuda.synchronize()
    lu_b, x_b, info_b = oracle.lu_factor_batched(db["At"].transpose(1, 2).cpu().numpy(), db["B"].cpu().numpy())
    lu_g = At.transpose(1, 2).cpu().numpy()
    x_g = Bt.transpose(1, 2).cpu().numpy()
    print(n, batch, "LU eq", np.array_equal(lu_g, lu_b), "x eq", np.array_equal(x_g, x_b), "info", info.tolist())
    d = np.abs(x_g - x_b)
    idx = np.argwhere(d > 0)
    print(" x mismatches", len(idx), idx[:10].tolist())
    print(" x_g", x_g[0, :8, 0], "\n x_o", x_b[0, :8, 0], "\n x_true", db["X"][0, :8, 0].cpu().numpy())
# oracle on CPU-generated inputs, nrhs 1 vs 2
for nr in (1, 2):
    dc = ebv_inputs.generate_batched(2, 32, seed=7, nrhs=nr)
    a = dc["At"].transpose(1, 2).numpy()
    b = dc["B"].numpy()
    _, xo, _ = oracle.lu_factor_batched(a, b)
    print("cpu-gen oracle nrhs", nr, np.abs(xo - dc["X"].numpy()).max(), b.shape, b.strides)
    dg = ebv_inputs.generate_batched(2, 32, seed=7, nrhs=nr, device=dev)
    a = dg["At"].transpose(1, 2).cpu().numpy()
    b = dg["B"].cpu().numpy()
    _, xo, _ = oracle.lu_factor_batched(a, b)
    print("gpu-gen oracle nrhs", nr, np.abs(xo - dg["X"].cpu().numpy()).max(), b.shape, b.strides, a.strides)
