"""Compact band storage on the GPU (ebv_lu_factor_band / ebv_lu_solve_band,
SURVEY §8f f4): the factors inside the band are bitwise the serial oracle's
on the dense matrix (Eq 6; no-pivot LU keeps the band, Golub & Van
Loan Thm 4.3.1), and the solution bitwise the oracle's solve (Eq 1,
P:31-33).  Large orders whose dense storage would not fit are checked by the
leading principal block (no pivoting: the LU of a leading block is the
leading block of the LU) and against the exact solution."""
import numpy as np
import pytest
import torch

import ebv_inputs
import oracle
import paper_1907_05767_b200 as ebv

pytestmark = pytest.mark.gpu


def bits_eq(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64), np.asarray(b, dtype=np.float64).view(np.uint64))


@pytest.fixture(scope="module")
def ctx():
    return ebv.Context(0)


def band_mask(n, kl, ku):
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    return ((i - j) <= kl) & ((j - i) <= ku)


@pytest.mark.parametrize("n,kl,ku,stencil", [(300, 17, 29, None), (1000, 64, 64, None), (777, 1, 1, None),
                                             (1500, 200, 3, None), (900, 30, 30, 30), (200, 199, 199, None)])
def test_band_factor_solve_bitwise(ctx, n, kl, ku, stencil):
    dev = torch.device("cuda:0")
    d = ebv_inputs.generate(n, seed=n + kl, device=dev, kl=kl, ku=ku, stencil_m=stencil)
    A = d["At"].T
    AB = ebv.band_pack(A, kl, ku)
    AB, info = ebv.lu_factor_band(AB, n, kl, ku, ctx=ctx)
    X = ebv.lu_solve_band(AB, d["B"], kl, ku, ctx=ctx)
    torch.cuda.synchronize()
    assert int(info) == 0
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    m = band_mask(n, kl, ku)
    lu_g = ebv.band_unpack(AB, n, kl, ku).cpu().numpy()
    assert bits_eq(lu_g[m], lu_o[m])
    assert (lu_o[~m] == 0).all()
    x_o = oracle.lu_solve(lu_o, d["B"].cpu().numpy())
    assert bits_eq(X.cpu().numpy(), x_o)


def test_band_equals_dense_storage_banded(ctx):
    n, kl, ku = 4096, 100, 37
    dev = torch.device("cuda:0")
    d = ebv_inputs.generate(n, seed=3, device=dev, kl=kl, ku=ku)
    A = d["At"].T
    LU, info = ebv.lu_factor_banded(A, kl, ku, ctx=ctx)
    AB, info2 = ebv.lu_factor_band(ebv.band_pack(A, kl, ku), n, kl, ku, ctx=ctx)
    torch.cuda.synchronize()
    assert int(info) == 0 and int(info2) == 0
    m = torch.from_numpy(band_mask(n, kl, ku)).to(dev)
    assert torch.equal(ebv.band_unpack(AB, n, kl, ku)[m].view(torch.int64), LU[m].view(torch.int64))


def test_band_large_order(ctx):
    """n = 131072 (dense storage would be 137 GB; band storage 0.5 GB)."""
    n, kl, ku, mlead = 131072, 128, 96, 1200
    dev = torch.device("cuda:0")
    ld = ebv.band_ld(kl, ku)
    g = ebv_inputs.generate_band(n, kl, ku, ebv.EBV_BAND_PAD, ld, seed=11, device=dev)
    AB = g["AB"]
    A_lead = ebv.band_unpack(AB[:mlead].contiguous(), mlead, kl, ku)   # leading principal block (same entries)
    AB, info = ebv.lu_factor_band(AB, n, kl, ku, ctx=ctx)
    X = ebv.lu_solve_band(AB, g["B"], kl, ku, ctx=ctx)
    torch.cuda.synchronize()
    assert int(info) == 0
    lu_o, _ = oracle.lu_factor(A_lead.cpu().numpy())
    m = band_mask(mlead, kl, ku)
    lu_g = ebv.band_unpack(AB[:mlead].contiguous(), mlead, kl, ku).cpu().numpy()
    assert bits_eq(lu_g[m], lu_o[m])
    err = (X - g["X"]).abs().max().item()
    assert err <= 1e-9, err


def test_band_argument_errors(ctx):
    dev = torch.device("cuda:0")
    info = torch.zeros((), dtype=torch.int64, device=dev)
    AB = torch.zeros(10, 64, dtype=torch.float64, device=dev)
    h = ctx.handle
    assert ebv.ebv_lu_factor_band(h, 10, 2, 2, AB.data_ptr(), 64, 0.0, info.data_ptr(), None) == 1   # ldab too small
    ld = ebv.band_ld(2, 2)
    AB = torch.zeros(10, ld, dtype=torch.float64, device=dev)
    assert ebv.ebv_lu_factor_band(h, 10, 2, 2, AB.data_ptr(), ld, -1.0, info.data_ptr(), None) == 1   # tau < 0
    assert ebv.ebv_lu_factor_band(h, 10, -1, 2, AB.data_ptr(), ld, 0.0, info.data_ptr(), None) == 1
