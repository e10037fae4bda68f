"""GPU parity of the chain-pipelined solve (k_solve2.cu; Eq 1).

ebv_lu_solve takes it for even n, even lda and 16-byte aligned factors (the
wavefront kernel of k_solve.cu otherwise).  Shapes span: fewer blocks than
the helpers' lag (n <= 384: the chain absorbs every tile), ragged last
blocks, several right-hand-side groups of 16, and the full C4 order, where
the oracle's substitution (O(n^2)) runs on the GPU's own factors.  All
comparisons are bitwise against the serial oracle."""
import numpy as np
import pytest
import torch

import ebv_inputs
import oracle

pytestmark = pytest.mark.gpu
ebv = pytest.importorskip("paper_1907_05767_b200")


def bits_eq(a, b):
    a = np.ascontiguousarray(np.asarray(a))
    b = np.ascontiguousarray(np.asarray(b))
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx(dev):
    return ebv.Context(0)


@pytest.mark.parametrize("n,nrhs", [(2, 1), (64, 1), (128, 2), (200, 1), (384, 1), (386, 3), (450, 16), (700, 1),
                                    (1000, 4), (2048, 1), (2050, 17), (4098, 5), (8192, 16), (3000, 33)])
def test_chain_solve_bitwise(dev, ctx, n, nrhs):
    d = ebv_inputs.generate(n, seed=7 * n + nrhs, nrhs=nrhs, device=dev)
    LU, info = ebv.lu_factor(d["At"].T, ctx=ctx)
    torch.cuda.synchronize()
    lu = LU.cpu().numpy()
    b = d["B"].cpu().numpy()
    x_o = oracle.lu_solve(lu, b)
    for _ in range(2):   # twice: the flag epochs advance per call
        X = ebv.lu_solve(LU, d["B"], ctx=ctx)
        torch.cuda.synchronize()
        assert bits_eq(X.cpu().numpy(), x_o)
    assert np.max(np.abs(x_o - d["X"].cpu().numpy())) <= 1e-10


@pytest.mark.parametrize("flavour", ebv_inputs.EDGE_FLAVOURS)
@pytest.mark.parametrize("force", [0, 1])
def test_chain_solve_edge_bitwise(dev, ctx, flavour, force):
    """Negative / mixed-sign / power-of-two-scaled pivots and subnormal or huge
    solutions; with EBV_DEBUG_FORCE_EXACT every backward block takes the
    redo path (true division, absorbers re-apply the block)."""
    n, nrhs = 1410, 3
    d = ebv_inputs.generate(n, seed=31, nrhs=nrhs, device=dev)
    A, B = ebv_inputs.edge_flavour(d["At"].T, d["B"], flavour, seed=31)
    LU, info = ebv.lu_factor(ebv.colmajor_copy(A), ctx=ctx)
    torch.cuda.synchronize()
    lu = LU.cpu().numpy()
    x_o = oracle.lu_solve(lu, B.cpu().numpy())
    ebv.set_debug(ebv.EBV_DEBUG_FORCE_EXACT if force else 0)
    try:
        X = ebv.lu_solve(LU, B.contiguous(), ctx=ctx)
        torch.cuda.synchronize()
    finally:
        ebv.set_debug(0)
    assert bits_eq(X.cpu().numpy(), x_o)


def test_chain_solve_full_c4(dev, ctx):
    """n = 32768 (BASELINE configs[3]), 1 RHS: the GPU solve on the GPU's
    factors equals the oracle's substitution on the same factors, bit for
    bit (the oracle's O(n^2) solve is feasible at this size)."""
    n = 32768
    d = ebv_inputs.generate(n, seed=1, nrhs=1, device=dev)
    LU, info = ebv.lu_factor(d["At"].T, ctx=ctx, inplace=False)
    del d["At"]
    X = ebv.lu_solve(LU, d["B"], ctx=ctx)
    torch.cuda.synchronize()
    x_g = X.cpu().numpy()
    lu = LU.cpu().numpy()
    del LU
    torch.cuda.empty_cache()
    x_o = oracle.lu_solve(lu, d["B"].cpu().numpy())
    assert bits_eq(x_g, x_o)
    assert np.max(np.abs(x_g - d["X"].cpu().numpy())) <= 1e-10
