"""The DMMA update variants and the leaf-solve knobs keep the
results bitwise.  Each knob is read when libebv.so loads, so every variant
runs in a child process: (1) ebv_update on integer-valued operands — every
product and partial sum is exact, so C - A B must equal the exact result for
any summation order; this pins the indexing of every tile path (ragged M,
N, K, odd leading dimensions, M <= 64); (2) factorizations at small orders
against the serial oracle bit for bit (Eq 6), which pins the
per-entry fma order through the variant."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import ebv_inputs, oracle
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
ctx = ebv.Context(0)
g = torch.Generator().manual_seed(7)
def cm(r, c, ld=None):
    ld = ld or r
    st = torch.randint(-8, 9, (c, ld), generator=g, dtype=torch.int64).to(torch.float64).to(dev)
    return st.T[:r, :]
for M, N, K, ldx in ((1, 1, 1, 0), (37, 29, 13, 3), (64, 300, 50, 0), (200, 130, 17, 1), (129, 65, 600, 2),
                     (1000, 70, 64, 0), (513, 257, 129, 5)):
    A = cm(M, K, M + ldx if ldx else None); B = cm(K, N, K + ldx if ldx else None); C = cm(M, N, M + ldx if ldx else None)
    ref = (C.cpu().numpy() - A.cpu().numpy() @ B.cpu().numpy())
    ebv.update(C, A, B, ctx=ctx)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), ref), (M, N, K, ldx)
def bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
for n, nb in ((700, 64), (1100, 128), (1300, 256)):
    d = ebv_inputs.generate(n, seed=n, device=dev)
    A = d["At"].T
    ctx.set_block(nb)
    LU, info = ebv.lu_factor(A, ctx=ctx)
    torch.cuda.synchronize()
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert bits(LU.cpu().numpy(), lu_o), (n, nb)
for n, kl, ku in ((600, 20, 33), (1000, 87, 5), (500, 3, 120)):
    d = ebv_inputs.generate(n, seed=n + kl, device=dev, kl=kl, ku=ku)
    A = d["At"].T
    LU, info = ebv.lu_factor_banded(A, kl, ku, ctx=ctx)
    torch.cuda.synchronize()
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert bits(LU.cpu().numpy(), lu_o), ("banded", n, kl, ku)
print("OK")
"""

VARIANTS = [
    {"EBV_GEMM_TMA": "-1"},   # cp.async kernel
    {"EBV_GEMM_TMA": "1"}, {"EBV_GEMM_TMA": "2"}, {"EBV_GEMM_TMA": "3"}, {"EBV_GEMM_TMA": "4"},
    {"EBV_GEMM_TMA": "5"}, {"EBV_GEMM_TMA": "6"}, {"EBV_GEMM_TMA": "7"},
    {"EBV_GEMM_CFG": "0"}, {"EBV_GEMM_CFG": "1"}, {"EBV_GEMM_CFG": "2"}, {"EBV_GEMM_CFG": "3"},
    {"EBV_TRSM_LLU_CC": "1", "EBV_U12_LA": "1"},
    {"EBV_PANEL_FUSED_ROWS": "0", "EBV_U12_SPLIT_ROWS": "100000"},
]


@pytest.mark.gpu
@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_bitwise(env):
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=dict(os.environ, **env), capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
