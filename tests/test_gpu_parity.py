"""GPU parity: the CUDA path through the C ABI against the serial oracle.

Bar: the path keeps the oracle's per-entry operation
order, so factor, solve and batched results are compared BITWISE
(np.array_equal) at sizes the oracle finishes in seconds — spanning several
leaves / tiles and ragged tails — and at the full BASELINE.json sizes via
properties that hold at any size (closed form, leading principal submatrix,
backward error).  The north_star tolerance (1e-10 relative, backward error
<= 1e-12) is asserted as well, as the documented fallback bar.
"""
import numpy as np
import pytest
import torch

import ebv_inputs
import oracle
from oracle import closed_form

def bits_eq(a, b):
    """Bitwise equality (IEEE bit patterns, so -0.0 != +0.0 and NaN payloads
    count), not just numeric equality."""
    a = np.ascontiguousarray(np.asarray(a))
    b = np.ascontiguousarray(np.asarray(b))
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.uint64), b.view(np.uint64))
    return np.array_equal(a, b)


pytestmark = pytest.mark.gpu

ebv = pytest.importorskip("paper_1907_05767_b200")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx(dev):
    return ebv.Context(0)


def run_factor(ctx, A, tau=0.0, path=ebv.EBV_PATH_BLOCKED, leaf=0, vector_ctas=0, nb=0):
    ctx.set_path(path)
    ctx.set_leaf(leaf)
    ctx.set_block(nb)
    ctx.set_vector_ctas(vector_ctas)
    LU, info = ebv.lu_factor(A, tau=tau, ctx=ctx)
    torch.cuda.synchronize()
    ctx.set_path(ebv.EBV_PATH_AUTO)
    ctx.set_leaf(0)
    ctx.set_block(0)
    ctx.set_vector_ctas(0)
    return LU.cpu().numpy(), int(info)


def tol_ok(g, o, rel=1e-10):
    m = np.max(np.abs(o)) if o.size else 0.0
    return np.max(np.abs(g - o)) <= rel * m if o.size else True


# ------------------------------------------------------------------ generator
def test_generator_device_equals_host(dev):
    c = ebv_inputs.generate(333, seed=4, nrhs=2)
    g = ebv_inputs.generate(333, seed=4, nrhs=2, device=dev)
    for k in ("At", "X", "B"):
        assert torch.equal(c[k], g[k].cpu())
    cb = ebv_inputs.generate_batched(50, 32, seed=4)
    gb = ebv_inputs.generate_batched(50, 32, seed=4, device=dev)
    for k in ("At", "X", "B"):
        assert torch.equal(cb[k], gb[k].cpu())


# ------------------------------------------------------------------ blocked factor
@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 33, 64, 65, 100, 129, 200, 257, 511, 1000, 1536])
def test_blocked_factor_bitwise(dev, ctx, n):
    d = ebv_inputs.generate(n, seed=n, device=dev)
    A = d["At"].T
    lu_g, info = run_factor(ctx, A)
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert info == info_o == 0
    assert bits_eq(lu_g, lu_o)


@pytest.mark.parametrize("nb,n", [(64, 700), (128, 700), (192, 700), (512, 700), (-1, 700), (64, 1537), (64, 3000)])
def test_blocked_schedules_bitwise(dev, ctx, nb, n):
    """(64, 1537/3000): many panel-leaf CTAs while the lookahead update occupies
    the GPU, so they start at different times (the diagonal block must not be
    overwritten before every CTA has read it)."""
    d = ebv_inputs.generate(n, seed=nb + 1000, device=dev)
    A = d["At"].T
    lu_g, _ = run_factor(ctx, A, nb=nb)
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert bits_eq(lu_g, lu_o)


@pytest.mark.parametrize("leaf", [8, 16, 24, 32, 48])
def test_blocked_factor_leaf_sizes_bitwise(dev, ctx, leaf):
    n = 300
    d = ebv_inputs.generate(n, seed=leaf, device=dev)
    A = d["At"].T
    lu_g, _ = run_factor(ctx, A, leaf=leaf)
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert bits_eq(lu_g, lu_o)


def test_blocked_factor_2048_bitwise_and_tolerance(dev, ctx):
    n = 2048
    d = ebv_inputs.generate(n, seed=21, device=dev)
    A = d["At"].T
    lu_g, _ = run_factor(ctx, A)
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert tol_ok(lu_g, lu_o)
    assert bits_eq(lu_g, lu_o)


def test_leading_dimension_and_odd_strides(dev, ctx):
    n, lda = 150, 173
    d = ebv_inputs.generate(n, seed=3, device=dev)
    store = torch.zeros(n, lda, dtype=torch.float64, device=dev)   # row j = column j, padded
    store[:, :n] = d["At"]
    A = store.T[:n, :]      # logical (n, n) with stride (1, lda)
    assert A.stride() == (1, lda)
    LU, info = ebv.lu_factor(A, ctx=ctx, inplace=True)
    torch.cuda.synchronize()
    lu_o, _ = oracle.lu_factor(d["At"].T.cpu().numpy())
    assert bits_eq(store.T[:n, :].cpu().numpy(), lu_o)
    assert not store[:, n:].any()      # padding untouched


def test_determinism(dev, ctx):
    d = ebv_inputs.generate(777, seed=5, device=dev)
    a, _ = run_factor(ctx, d["At"].T)
    b, _ = run_factor(ctx, d["At"].T)
    assert bits_eq(a, b)


# ------------------------------------------------------------------ pivots / info
def test_info_zero_pivot_and_tau(dev, ctx):
    n = 130
    for k0 in (0, 63, 64, 100, 129):
        A = torch.eye(n, dtype=torch.float64, device=dev) * 2.0
        A[k0, k0] = 0.0
        _, info = run_factor(ctx, A)
        assert info == k0 + 1
        _, info_v = run_factor(ctx, A, path=ebv.EBV_PATH_VECTOR)
        assert info_v == k0 + 1
    A = torch.eye(n, dtype=torch.float64, device=dev)
    A[5, 5] = 1e-30
    assert run_factor(ctx, A, tau=0.0)[1] == 0
    assert run_factor(ctx, A, tau=1e-20)[1] == 6
    assert run_factor(ctx, A, tau=-1.0)[1] == 6      # default n*eps*||A||_inf
    # first failing step wins, the factorization continues
    A = torch.eye(n, dtype=torch.float64, device=dev)
    A[70, 70] = 0.0
    A[3, 3] = 0.0
    assert run_factor(ctx, A)[1] == 4


def test_argument_errors(dev, ctx):
    L = ebv.lib()
    info = torch.zeros((), dtype=torch.int64, device=dev)
    A = torch.zeros(4, 4, dtype=torch.float64, device=dev)
    assert L.ebv_lu_factor(ctx.handle, -1, A.data_ptr(), 4, 0.0, info.data_ptr(), None) == 1
    assert L.ebv_lu_factor(ctx.handle, 4, A.data_ptr(), 3, 0.0, info.data_ptr(), None) == 1
    assert L.ebv_lu_factor(ctx.handle, 4, None, 4, 0.0, info.data_ptr(), None) == 1
    assert L.ebv_lu_factor(ctx.handle, 0, None, 1, 0.0, info.data_ptr(), None) == 0
    assert L.ebv_lu_solve(ctx.handle, 4, A.data_ptr(), 4, None, 4, 1, None) == 1
    assert L.ebv_lu_factor_batched(ctx.handle, 513, A.data_ptr(), 513, 513 * 513, 1, None, 513, 0, 0, 0.0,
                                   info.data_ptr(), None) == 5
    torch.cuda.synchronize()


# ------------------------------------------------------------------ solve
@pytest.mark.parametrize("n,nrhs", [(1, 1), (5, 2), (64, 1), (65, 3), (200, 16), (333, 17), (1000, 1), (1536, 5)])
def test_solve_bitwise(dev, ctx, n, nrhs):
    d = ebv_inputs.generate(n, seed=100 + n, nrhs=nrhs, device=dev)
    A = d["At"].T
    LU, _ = ebv.lu_factor(A, ctx=ctx)
    X = ebv.lu_solve(LU, d["B"], ctx=ctx)
    torch.cuda.synchronize()
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    x_o = oracle.lu_solve(lu_o, d["B"].cpu().numpy())
    assert bits_eq(X.cpu().numpy(), x_o)
    assert np.max(np.abs(X.cpu().numpy() - d["X"].cpu().numpy())) <= 1e-10


def test_solve_vector_rhs_and_backward_error(dev, ctx):
    n = 4096
    d = ebv_inputs.generate(n, seed=9, nrhs=1, device=dev)
    A = d["At"].T
    LU, _ = ebv.lu_factor(A, ctx=ctx)
    x = ebv.lu_solve(LU, d["B"][:, 0], ctx=ctx)
    torch.cuda.synchronize()
    r = (A @ x - d["B"][:, 0]).abs().max() / (A.abs().sum(1).max() * x.abs().max())
    assert float(r) <= 1e-12


def test_block_width_query(dev):
    c = ebv.Context(0)
    assert c.block_width(1024) == 64 and c.block_width(8192) == 128
    assert c.block_width(16384) == 256 and c.block_width(32768) == 512
    c.set_block(192)
    assert c.block_width(32768) == 192
    c.set_block(-1)
    assert c.block_width(1000) == -1


@pytest.mark.parametrize("n,nrhs", [(700, 64), (700, 16), (700, 17), (1537, 100), (129, 300), (64, 65), (333, 2)])
def test_solve_many_rhs_bitwise(dev, ctx, n, nrhs):
    """Up to 64 columns: interleaved wavefront chains; more: recursive TRSM
    with DMMA updates — both bitwise the oracle's substitutions."""
    d = ebv_inputs.generate(n, seed=n + nrhs, nrhs=nrhs, device=dev)
    A = d["At"].T
    LU, info = ebv.lu_factor(A, ctx=ctx)
    X = ebv.lu_solve(LU, d["B"], ctx=ctx)
    torch.cuda.synchronize()
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert bits_eq(LU.cpu().numpy(), lu_o)
    assert bits_eq(X.cpu().numpy(), oracle.lu_solve(lu_o, d["B"].cpu().numpy()))


# ------------------------------------------------------------------ left-looking / host-resident
@pytest.mark.parametrize("n,nb", [(1, 0), (64, 0), (65, 64), (700, 64), (700, 128), (1537, 64), (3000, 0),
                                  (2100, 256)])
def test_left_looking_bitwise(dev, ctx, n, nb):
    d = ebv_inputs.generate(n, seed=n + 77, device=dev)
    A = d["At"].T
    c = ebv.Context(0, path=ebv.EBV_PATH_LEFT)
    c.set_block(nb)
    LU, info = ebv.lu_factor(A, ctx=c)
    torch.cuda.synchronize()
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert int(info) == info_o
    assert bits_eq(LU.cpu().numpy(), lu_o)


@pytest.mark.parametrize("n,pinned,tau", [(700, True, 0.0), (1537, False, 0.0), (3000, True, 0.0), (513, True, -1.0),
                                          (16384, True, 0.0)])
def test_factor_host_bitwise(dev, ctx, n, pinned, tau):
    """ebv_lu_factor_host: the matrix streamed from host memory block by block
    under the left-looking factorization — bitwise the oracle."""
    d = ebv_inputs.generate(n, seed=n + 78)
    hA = d["At"].T                      # CPU, column-major storage
    if pinned:
        hA = hA.mT.contiguous().pin_memory().mT
    LU, info = ebv.lu_factor_host(hA, tau=tau, ctx=ctx)
    cl = ebv.Context(0, path=ebv.EBV_PATH_LEFT)          # the streamed (left-looking) form
    LU2, info2 = ebv.lu_factor_host(hA, tau=tau, ctx=cl)
    torch.cuda.synchronize()
    assert bits_eq(LU2.cpu().numpy(), LU.cpu().numpy()) and int(info2) == int(info)
    if n > 4096:   # the streamed right-looking form: compare with the device factorization (same bits)
        LUd, infod = ebv.lu_factor(d["At"].T.to(dev), ctx=ctx)
        torch.cuda.synchronize()
        assert int(info) == int(infod) == 0
        assert torch.equal(LU.view(torch.int64), LUd.view(torch.int64))
        lead = 1024   # and the leading block with the oracle (the same computation)
        lu_o, _ = oracle.lu_factor(d["At"].T.numpy()[:lead, :lead])
        assert bits_eq(LU[:lead, :lead].cpu().numpy(), lu_o)
        return
    lu_o, info_o = oracle.lu_factor(d["At"].T.numpy(), tau=(n * np.finfo(float).eps *
                                                            np.abs(d["At"].T.numpy()).sum(1).max()) if tau < 0 else 0.0)
    assert int(info) == info_o
    assert bits_eq(LU.cpu().numpy(), lu_o)


# ------------------------------------------------------------------ f4: banded / stencil (zero-skip)
@pytest.mark.parametrize("n,kl,ku,stencil", [(700, 30, 50, 0), (1537, 200, 64, 0), (3000, 1, 600, 0),
                                             (64 * 64, 64, 64, 64), (5, 1, 1, 0), (1000, 0, 0, 0)])
def test_banded_bitwise(dev, ctx, n, kl, ku, stencil):
    """Zero-skip banded factor + solve equal the dense oracle bitwise (the
    band is preserved; entries outside it stay exactly zero)."""
    if stencil:
        d = ebv_inputs.generate(n, seed=n, nrhs=2, device=dev, stencil_m=stencil)
    else:
        d = ebv_inputs.generate(n, seed=n + kl, nrhs=2, device=dev, kl=kl, ku=ku)
    A = d["At"].T
    LU, info = ebv.lu_factor_banded(A, kl, ku, ctx=ctx)
    X = ebv.lu_solve_banded(LU, d["B"], kl, ku, ctx=ctx)
    torch.cuda.synchronize()
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert int(info) == info_o == 0
    assert bits_eq(LU.cpu().numpy(), lu_o)
    assert bits_eq(X.cpu().numpy(), oracle.lu_solve(lu_o, d["B"].cpu().numpy()))


# ------------------------------------------------------------------ f3: unit diagonal, LDU
@pytest.mark.parametrize("n,nrhs", [(1, 1), (2, 0), (300, 3), (1537, 1)])
def test_normalize_unit_diagonal_bitwise(dev, ctx, n, nrhs):
    d = ebv_inputs.generate(n, seed=n + 5, nrhs=max(nrhs, 1), device=dev)
    A = d["At"].T
    B = d["B"] if nrhs else None
    An, Bn, scales, info = ebv.normalize_unit_diagonal(A, B, ctx=ctx)
    torch.cuda.synchronize()
    a_o, b_o, s_o, info_o = oracle.normalize_unit_diagonal(A.cpu().numpy(), B.cpu().numpy() if nrhs else None)
    assert int(info) == info_o == 0
    assert bits_eq(An.cpu().numpy(), a_o)
    assert bits_eq(scales.cpu().numpy(), s_o)
    if nrhs:
        assert bits_eq(Bn.cpu().numpy(), b_o)
    # the normalized system is factored and solved like any other (Eq 2 shape)
    LU, inf2 = ebv.lu_factor(An, ctx=ctx)
    torch.cuda.synchronize()
    assert int(inf2) == 0 and bits_eq(LU.cpu().numpy(), oracle.lu_factor(a_o)[0])


def test_normalize_zero_diagonal_reported(dev, ctx):
    A = torch.eye(5, dtype=torch.float64, device=dev) * 2.0
    A[3, 3] = 0.0
    A[4, 4] = 0.0
    An, _, scales, info = ebv.normalize_unit_diagonal(A, None, ctx=ctx)
    torch.cuda.synchronize()
    assert int(info) == 4
    assert scales[3].item() == 0.0 and An[3, 3].item() == 0.0 and An[0, 0].item() == 1.0


@pytest.mark.parametrize("n", [1, 2, 65, 700, 3000])
def test_lu_to_ldu_bitwise(dev, ctx, n):
    d = ebv_inputs.generate(n, seed=n + 9, device=dev)
    LU, _ = ebv.lu_factor(d["At"].T, ctx=ctx)
    LDU, D = ebv.lu_to_ldu(LU, ctx=ctx)
    torch.cuda.synchronize()
    ldu_o, d_o = oracle.lu_to_ldu(LU.cpu().numpy())
    assert bits_eq(LDU.cpu().numpy(), ldu_o)
    assert bits_eq(D.cpu().numpy(), d_o)


# ------------------------------------------------------------------ vector path (EbV owner map)
@pytest.mark.parametrize("n,ctas", [(1, 0), (2, 0), (3, 0), (64, 0), (255, 0), (1024, 0), (1024, 128), (1024, -128),
                                    (1000, 100), (1536, 0), (300, -7), (301, 5), (33, 1)])
def test_vector_path_bitwise(dev, ctx, n, ctas):
    d = ebv_inputs.generate(n, seed=3 * n + 1, device=dev)
    A = d["At"].T
    lu_g, info = run_factor(ctx, A, path=ebv.EBV_PATH_VECTOR, vector_ctas=ctas)
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert info == info_o
    assert bits_eq(lu_g, lu_o)


# ------------------------------------------------------------------ batched
@pytest.mark.parametrize("n,batch,nrhs", [(32, 1000, 1), (32, 1, 1), (32, 7, 2), (1, 5, 1), (7, 33, 3),
                                          (31, 64, 16), (32, 257, 0), (33, 50, 1), (48, 31, 3), (64, 200, 1),
                                          (64, 3, 16), (64, 9, 0),
                                          (65, 9, 1), (100, 20, 3), (128, 7, 16), (200, 5, 2), (511, 3, 1), (512, 2, 4)])
def test_batched_bitwise(dev, ctx, n, batch, nrhs):
    db = ebv_inputs.generate_batched(batch, n, seed=n + batch, nrhs=max(nrhs, 1), device=dev)
    At = db["At"].clone()
    Bt = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)[:, :nrhs] if nrhs else None
    if Bt is not None:
        Bt = Bt.contiguous()
    info = ebv.lu_factor_batched(At, Bt, ctx=ctx)
    torch.cuda.synchronize()
    a = db["At"].transpose(1, 2).cpu().numpy()
    b = db["B"][:, :, :nrhs].cpu().numpy() if nrhs else None
    lu_o, x_o, info_o = oracle.lu_factor_batched(a, b)
    assert bits_eq(info.cpu().numpy(), info_o)
    assert bits_eq(At.transpose(1, 2).cpu().numpy(), lu_o)
    if nrhs:
        assert bits_eq(Bt.transpose(1, 2).cpu().numpy(), x_o)


@pytest.mark.parametrize("n,batch,nrhs", [(32, 1000, 1), (32, 333, 16), (7, 65, 3), (1, 4, 2), (31, 2, 5),
                                          (64, 100, 2), (40, 7, 1), (130, 6, 3), (300, 3, 16)])
def test_batched_solve_only_bitwise(dev, ctx, n, batch, nrhs):
    """Factor once, solve many: ebv_lu_solve_batched on the
    factors of ebv_lu_factor_batched equals the oracle's solve of every
    system bitwise, for two different right-hand-side sets, and leaves LU
    untouched."""
    db = ebv_inputs.generate_batched(batch, n, seed=3 * n + batch, nrhs=nrhs, device=dev)
    LUt = db["At"].clone()
    info = ebv.lu_factor_batched(LUt, None, ctx=ctx)
    torch.cuda.synchronize()
    assert not info.any().item()
    lu_before = LUt.clone()
    a = db["At"].transpose(1, 2).cpu().numpy()
    lu_o = np.stack([oracle.lu_factor(a[s])[0] for s in range(batch)])
    assert bits_eq(LUt.transpose(1, 2).cpu().numpy(), lu_o)
    for rhs_seed in (0, 1):
        B = db["B"] if rhs_seed == 0 else torch.flip(db["B"], dims=[1]) * 0.5
        Bt = B.transpose(1, 2).clone(memory_format=torch.contiguous_format)
        ebv.lu_solve_batched(LUt, Bt, ctx=ctx)
        torch.cuda.synchronize()
        b = B.cpu().numpy()
        x_o = np.stack([oracle.lu_solve(lu_o[s], b[s]) for s in range(batch)])
        assert bits_eq(Bt.transpose(1, 2).cpu().numpy(), x_o)
    assert torch.equal(LUt, lu_before)


def test_batched_full_size_c5(dev, ctx):
    """BASELINE.json configs[4]: 100k systems of n = 32, every system bitwise."""
    batch = 100_000
    db = ebv_inputs.generate_batched(batch, 32, seed=1, nrhs=1, device=dev)
    At = db["At"].clone()
    Bt = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
    info = ebv.lu_factor_batched(At, Bt, ctx=ctx)
    torch.cuda.synchronize()
    lu_o, x_o, info_o = oracle.lu_factor_batched(db["At"].transpose(1, 2).cpu().numpy(), db["B"].cpu().numpy())
    assert not info.any().item()
    assert bits_eq(At.transpose(1, 2).cpu().numpy(), lu_o)
    assert bits_eq(Bt.transpose(1, 2).cpu().numpy(), x_o)


def test_batched_singular_systems(dev, ctx):
    db = ebv_inputs.generate_batched(10, 32, seed=2, device=dev)
    At = db["At"].clone()
    At[3, 5, :] = 0.0            # column 5 of system 3 zero -> u_55 == 0 exactly
    At[7, 0, 0] = 0.0            # first pivot of system 7
    ref = At.transpose(1, 2).cpu().numpy().copy()
    info = ebv.lu_factor_batched(At, None, ctx=ctx)
    torch.cuda.synchronize()
    _, _, info_o = oracle.lu_factor_batched(ref, None)
    assert info.cpu().tolist() == info_o.tolist()
    assert info_o[3] == 6 and info_o[7] == 1


# ------------------------------------------------------------------ full-size properties (C3 / C4)
def test_closed_form_full_size(dev, ctx):
    """A = n I + s s^T at BASELINE's n = 32768: every one of the n^2 entries
    of the GPU factor against the closed form (oracle/closed_form.py)."""
    n = 32768
    At, s = ebv_inputs.closed_form_inputs(n, seed=1, device=dev)
    A = At.T  # symmetric anyway
    LU, info = ebv.lu_factor(A, ctx=ctx, inplace=False)
    torch.cuda.synchronize()
    assert int(info) == 0
    del A, At
    d, cl, cu = closed_form.factors_exact(n, n, 1, s.cpu().numpy())
    dv = torch.tensor([float(x) for x in d], dtype=torch.float64, device=dev)
    clv = torch.tensor([float(x) for x in cl], dtype=torch.float64, device=dev)
    cuv = torch.tensor([float(x) for x in cu], dtype=torch.float64, device=dev)
    sf = s.to(torch.float64)
    worst = 0.0
    for j0 in range(0, n, 2048):
        j1 = j0 + 2048
        blk = LU[:, j0:j1]                                  # (n, 2048)
        rows = torch.arange(n, device=dev)[:, None]
        cols = torch.arange(j0, j1, device=dev)[None, :]
        ss = sf[:, None] * sf[None, j0:j1]
        ref = torch.where(rows > cols, ss * clv[None, j0:j1],
                          torch.where(rows < cols, ss * cuv[:, None], dv[None, j0:j1].expand(n, -1)))
        rel = ((blk - ref).abs() / ref.abs()).max().item()
        worst = max(worst, rel)
    assert worst <= 1e-12, worst


def test_c3_n8192_leading_submatrix_and_backward_error(dev, ctx):
    """configs[2]: n = 8192, 16 right-hand sides.  LU of the leading 1536 x 1536
    principal submatrix equals the oracle bitwise (it is the same computation);
    full solve: x vs the exact x_true and the backward error bound."""
    n, m = 8192, 1536
    d = ebv_inputs.generate(n, seed=2, nrhs=16, device=dev)
    A = d["At"].T
    LU, info = ebv.lu_factor(A, ctx=ctx)
    X = ebv.lu_solve(LU, d["B"], ctx=ctx)
    torch.cuda.synchronize()
    lu_o, _ = oracle.lu_factor(A[:m, :m].cpu().numpy())
    assert bits_eq(LU[:m, :m].cpu().numpy(), lu_o)
    assert (X - d["X"]).abs().max().item() <= 1e-10
    r = ((A @ X - d["B"]).abs().max() / (A.abs().sum(1).max() * X.abs().max())).item()
    assert r <= 1e-12


def test_c4_n32768_properties(dev, ctx):
    """configs[3] size on one GPU: leading principal 1024 block bitwise vs the
    oracle, sampled reconstruction (LU)_ij == a_ij within the backward-error
    bound, and x vs the exact solution."""
    n, m = 32768, 1024
    d = ebv_inputs.generate(n, seed=1, nrhs=1, device=dev)
    A = d["At"].T
    LU, info = ebv.lu_factor(A, ctx=ctx)
    x = ebv.lu_solve(LU, d["B"][:, 0], ctx=ctx)
    torch.cuda.synchronize()
    assert int(info) == 0
    lu_o, _ = oracle.lu_factor(A[:m, :m].cpu().numpy())
    assert bits_eq(LU[:m, :m].cpu().numpy(), lu_o)
    assert (x - d["X"][:, 0]).abs().max().item() <= 1e-10
    g = torch.Generator(device="cpu").manual_seed(0)
    ii = torch.randint(0, n, (2000,), generator=g).tolist()
    jj = torch.randint(0, n, (2000,), generator=g).tolist()
    amax = A.abs().max().item()
    for i, j in zip(ii, jj):
        if i <= j:   # (LU)_ij = sum_{p<i} l_ip u_pj + u_ij
            v = (LU[i, :i] * LU[:i, j]).sum() + LU[i, j]
        else:        # (LU)_ij = sum_{p<j} l_ip u_pj + l_ij u_jj
            v = (LU[i, :j] * LU[:j, j]).sum() + LU[i, j] * LU[j, j]
        assert abs(v.item() - A[i, j].item()) <= 1e-12 * amax


def test_graph_replay_bitwise(dev, ctx):
    """The second identical call captures a CUDA Graph, later calls replay it:
    every result bitwise equal to the oracle; launch accounting continues."""
    n = 1100
    d = ebv_inputs.generate(n, seed=31, device=dev)
    lu_o, _ = oracle.lu_factor(d["At"].T.cpu().numpy())
    Aw = torch.empty_like(d["At"])
    info = torch.zeros((), dtype=torch.int64, device=dev)
    s = torch.cuda.Stream()
    counts = []
    with torch.cuda.stream(s):
        for rep in range(4):
            Aw.copy_(d["At"])
            c0 = ctx.launch_count()
            st = ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), s.cuda_stream)
            assert st == 0, ebv.ebv_last_error()
            counts.append(ctx.launch_count() - c0)
            s.synchronize()
            assert bits_eq(Aw.T.cpu().numpy(), lu_o), rep
            assert int(info) == 0
    assert counts[0] == counts[2] == counts[3] > 10


# ------------------------------------------------------------------ randomized schedule stress
_RNG_CASES = []
_rs = np.random.default_rng(20261018)
for _ in range(14):
    _n = int(_rs.integers(1, 1400))
    _RNG_CASES.append((_n, int(_rs.choice([0, 64, 128, 192, 256, -1])), int(_rs.choice([8, 16, 32, 64])),
                       int(_rs.choice([ebv.EBV_PATH_BLOCKED, ebv.EBV_PATH_LEFT])), bool(_rs.integers(0, 2)),
                       int(_rs.integers(1, 70))))


@pytest.mark.parametrize("n,nb,leaf,path,la,nrhs", _RNG_CASES)
def test_random_schedules_bitwise(dev, n, nb, leaf, path, la, nrhs):
    """Random sizes x block widths x leaf sizes x schedules x lookahead x
    right-hand-side counts: factors and solutions bitwise the oracle's."""
    c = ebv.Context(0, path=path)
    c.set_leaf(leaf)
    if nb > 0:
        nb = max(leaf, (nb // leaf) * leaf)
    c.set_block(nb if path == ebv.EBV_PATH_BLOCKED or nb >= 0 else 0)
    c.set_lookahead(la)
    d = ebv_inputs.generate(n, seed=n * 7 + nrhs, nrhs=nrhs, device=dev)
    A = d["At"].T
    LU, info = ebv.lu_factor(A, ctx=c)
    X = ebv.lu_solve(LU, d["B"], ctx=c)
    torch.cuda.synchronize()
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert int(info) == info_o == 0
    assert bits_eq(LU.cpu().numpy(), lu_o)
    assert bits_eq(X.cpu().numpy(), oracle.lu_solve(lu_o, d["B"].cpu().numpy()))


@pytest.mark.parametrize("n,tau", [(100, 0.0), (150, -1.0), (300, 0.25)])
def test_batched_medium_info(dev, ctx, n, tau):
    """Batched medium orders: per-system info (first failing
    1-based step, reading R9's threshold) equals the oracle's, including
    tau < 0 (n * eps * ||A_s||_inf per system), and the factors stay bitwise."""
    batch = 5
    db = ebv_inputs.generate_batched(batch, n, seed=n, nrhs=1, device=dev)
    At = db["At"].clone()
    At[2, 0, 0] = 0.0                      # system 2: a zero first pivot
    At[4, 70, 70] = 1e-300                 # system 4: a tiny pivot at step 71 (caught by tau < 0 / tau > 0)
    a = At.transpose(1, 2).cpu().numpy()
    info = ebv.lu_factor_batched(At, None, tau=tau, ctx=ctx)
    torch.cuda.synchronize()
    if tau >= 0:
        lu_o, _, info_o = oracle.lu_factor_batched(a, None, tau=tau)
    else:   # the API's default floor per system (reading R9), passed to the oracle explicitly
        res = [oracle.lu_factor(a[s], n * 2.220446049250313e-16 * np.abs(a[s]).sum(1).max()) for s in range(batch)]
        lu_o = np.stack([r[0] for r in res])
        info_o = np.array([r[1] for r in res], dtype=np.int32)
    assert bits_eq(info.cpu().numpy(), info_o)
    assert info_o[2] == 1
    ok = [s for s in range(batch) if info_o[s] == 0]
    assert bits_eq(At.transpose(1, 2).cpu().numpy()[ok], lu_o[ok])


@pytest.mark.parametrize("n", [700, 16384])
def test_stream_wait_host_copy(dev, ctx, n):
    """ebv_stream_wait_host_copy orders another stream after the library's
    host stream-in (copy-first path for n = 700, streamed right-looking path
    for n = 16384); the factors stay bitwise those of the device path."""
    d = ebv_inputs.generate(n, seed=5, device=dev, with_b=False)
    hA = torch.empty(d["At"].shape, dtype=torch.float64, pin_memory=True)
    hA.copy_(d["At"])
    A = torch.empty_like(d["At"])
    A2 = torch.empty_like(d["At"])
    info = torch.zeros((), dtype=torch.int64, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    assert ebv.ebv_lu_factor_host(ctx.handle, n, hA.data_ptr(), n, A.data_ptr(), n, 0.0, info.data_ptr(),
                                  s1.cuda_stream) == 0
    assert ebv.ebv_stream_wait_host_copy(ctx.handle, s2.cuda_stream) == 0
    with torch.cuda.stream(s2):
        A2.copy_(hA, non_blocking=True)
    torch.cuda.synchronize()
    assert int(info) == 0
    ref, _ = run_factor(ctx, d["At"].T.clone())
    assert bits_eq(A.T.cpu().numpy(), ref)
    assert torch.equal(A2, d["At"])
