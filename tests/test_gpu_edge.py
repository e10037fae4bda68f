"""GPU parity on the method's sign and scale edge cases (Eq 6-a's division,
P:67; Eq 1's substitutions).

The generated systems (all-positive pivots) are transformed exactly
(ebv_inputs.edge_flavour: negation, row / column sign flips, power-of-two
row and column scalings up to 2^+-500, right-hand sides scaled so the
solution is subnormal or huge), which gives negative and mixed-sign pivots
and multipliers / quotients far outside the range the kernels' fast
verified-quotient division accepts.  Every path is compared BITWISE (IEEE
bit patterns) with the serial oracle on the same inputs, once as shipped and
once with EBV_DEBUG_FORCE_EXACT, which sends every verified-quotient step to
its redo-with-true-division branch (those branches must give the same bits).
"""
import numpy as np
import pytest
import torch

import ebv_inputs
import oracle

pytestmark = pytest.mark.gpu
ebv = pytest.importorskip("paper_1907_05767_b200")

FLAVOURS = ebv_inputs.EDGE_FLAVOURS


def bits_eq(a, b):
    a = np.ascontiguousarray(np.asarray(a))
    b = np.ascontiguousarray(np.asarray(b))
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.uint64), b.view(np.uint64))
    return np.array_equal(a, b)


def first_diff(a, b):
    a, b = np.asarray(a), np.asarray(b)
    bad = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
    return f"{len(bad)} entries differ; first {bad[:3].tolist()}: {a[tuple(bad[0])]!r} vs {b[tuple(bad[0])]!r}" \
        if len(bad) else "equal"


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx(dev):
    return ebv.Context(0)


@pytest.fixture(params=[0, ebv.EBV_DEBUG_FORCE_EXACT], ids=["fast", "force_exact"])
def force(request, dev):
    ebv.set_debug(request.param)
    yield request.param
    ebv.set_debug(0)


def system(n, seed, nrhs, flavour, dev):
    d = ebv_inputs.generate(n, seed=seed, nrhs=nrhs, device=dev)
    A, B = ebv_inputs.edge_flavour(d["At"].T, d["B"], flavour, seed=seed)
    return ebv.colmajor_copy(A), B.contiguous()


def check_factor_solve(ctx, A, B, path=ebv.EBV_PATH_AUTO, nb=0):
    ctx.set_path(path)
    ctx.set_block(nb)
    try:
        LU, info = ebv.lu_factor(A, ctx=ctx)
        X = ebv.lu_solve(LU, B, ctx=ctx)
        torch.cuda.synchronize()
    finally:
        ctx.set_path(ebv.EBV_PATH_AUTO)
        ctx.set_block(0)
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert int(info) == info_o == 0
    lu_g = LU.cpu().numpy()
    assert bits_eq(lu_g, lu_o), first_diff(lu_g, lu_o)
    x_o = oracle.lu_solve(lu_o, B.cpu().numpy())
    x_g = X.cpu().numpy()
    assert bits_eq(x_g, x_o), first_diff(x_g, x_o)


@pytest.mark.parametrize("flavour", FLAVOURS)
@pytest.mark.parametrize("n,nrhs,nb", [(700, 1, 0), (1537, 3, 128), (1538, 3, 128), (333, 16, -1), (334, 16, 0)])
def test_blocked_edge_bitwise(dev, ctx, force, flavour, n, nrhs, nb):
    """Blocked (panel leaf, U12 leaf solve, DMMA update) and the recursive
    schedule; wavefront solve with 1 / 3 / 16 right-hand sides."""
    A, B = system(n, n + nrhs, nrhs, flavour, dev)
    check_factor_solve(ctx, A, B, nb=nb)


@pytest.mark.parametrize("flavour", FLAVOURS)
def test_trsm_solve_edge_bitwise(dev, ctx, force, flavour):
    """Many right-hand sides (the recursive TRSM + DMMA solve path)."""
    A, B = system(300, 41, 150, flavour, dev)
    check_factor_solve(ctx, A, B)


@pytest.mark.parametrize("flavour", FLAVOURS)
@pytest.mark.parametrize("n", [1024, 301])
def test_vector_path_edge_bitwise(dev, ctx, force, flavour, n):
    A, B = system(n, n, 1, flavour, dev)
    check_factor_solve(ctx, A, B, path=ebv.EBV_PATH_VECTOR)


@pytest.mark.parametrize("flavour", FLAVOURS)
@pytest.mark.parametrize("n,batch,nrhs", [(32, 500, 1), (32, 64, 16), (20, 40, 2), (20, 41, 1), (32, 33, 0),
                                          (64, 60, 1), (200, 4, 3)])
def test_batched_edge_bitwise(dev, ctx, force, flavour, n, batch, nrhs):
    """n = 32 (lane-paired kernels: 1 RHS — forward fused into the factor,
    Markstein backward with the deferred test — and 16 RHS), n = 20
    (padding; 1 and 2 RHS), factor only (nrhs = 0), n = 64 (CTA per
    system), n = 200 (the batched blocked schedule)."""
    db = ebv_inputs.generate_batched(batch, n, seed=n + batch + nrhs, nrhs=max(nrhs, 1), device=dev)
    A = db["At"].transpose(1, 2)                    # logical (batch, n, n)
    A2, B2 = ebv_inputs.edge_flavour(A, db["B"], flavour, seed=n)
    a_np, b_np = A2.cpu().numpy().copy(), B2.cpu().numpy().copy()   # before the in-place factorization
    At = A2.transpose(1, 2).clone(memory_format=torch.contiguous_format)
    Bt = B2.transpose(1, 2).clone(memory_format=torch.contiguous_format) if nrhs else None
    info = ebv.lu_factor_batched(At, Bt, ctx=ctx)
    torch.cuda.synchronize()
    lu_o, x_o, info_o = oracle.lu_factor_batched(a_np, b_np if nrhs else None)
    assert bits_eq(info.cpu().numpy(), info_o)
    lu_g = At.transpose(1, 2).cpu().numpy()
    assert bits_eq(lu_g, lu_o), first_diff(lu_g, lu_o)
    if not nrhs:
        return
    x_g = Bt.transpose(1, 2).cpu().numpy()
    assert bits_eq(x_g, x_o), first_diff(x_g, x_o)
    # solve-only on the factors (RG > 1 chains for 16 RHS)
    Bt2 = torch.from_numpy(b_np).to(dev).transpose(1, 2).clone(memory_format=torch.contiguous_format)
    ebv.lu_solve_batched(At, Bt2, ctx=ctx)
    torch.cuda.synchronize()
    assert bits_eq(Bt2.transpose(1, 2).cpu().numpy(), x_o)


@pytest.mark.parametrize("flavour", FLAVOURS)
def test_dist_emulated_edge_bitwise(dev, ctx, force, flavour):
    n, nb, P, nrhs = 700, 64, 3, 2
    A, B = system(n, 5, nrhs, flavour, dev)
    At = A.T                                   # (n, n) storage rows = columns (A column-major)
    slabs, colmaps = [], []
    for r in range(P):
        cols = ebv.dist_local_columns(n, nb, r, P, 0)
        slabs.append(At[torch.tensor(cols, dtype=torch.long, device=dev)].clone())
        colmaps.append(cols)
    info = torch.zeros((), dtype=torch.int64, device=dev)
    sh = torch.cuda.current_stream().cuda_stream
    assert ebv.ebv_lu_factor_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n, 0.0,
                                           info.data_ptr(), sh) == 0, ebv.ebv_last_error()
    Bc = B.T.contiguous()
    assert ebv.ebv_lu_solve_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n,
                                          Bc.data_ptr(), n, nrhs, sh) == 0, ebv.ebv_last_error()
    torch.cuda.synchronize()
    full = np.zeros((n, n))
    for st, cols in zip(slabs, colmaps):
        full[:, cols] = st.T.cpu().numpy()
    lu_o, info_o = oracle.lu_factor(A.cpu().numpy())
    assert int(info) == info_o == 0
    assert bits_eq(full, lu_o), first_diff(full, lu_o)
    x_o = oracle.lu_solve(lu_o, B.cpu().numpy())
    assert bits_eq(Bc.T.cpu().numpy(), x_o)


def test_forced_exact_really_redoes(dev, ctx):
    """The knob is live: with EBV_DEBUG_FORCE_EXACT the batched n = 32 kernel
    takes its true-division branch (slower), and the bits do not change."""
    db = ebv_inputs.generate_batched(20000, 32, seed=9, nrhs=16, device=dev)
    LUt = db["At"].clone()
    ebv.lu_factor_batched(LUt, None, ctx=ctx)
    times = {}
    outs = {}
    for flag in (0, ebv.EBV_DEBUG_FORCE_EXACT):
        ebv.set_debug(flag)
        try:
            for rep in range(3):
                Bt = db["B"].transpose(1, 2).contiguous()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ebv.lu_solve_batched(LUt, Bt, ctx=ctx)
                e1.record()
                torch.cuda.synchronize()
                times[flag] = min(times.get(flag, 1e9), e0.elapsed_time(e1))
            outs[flag] = Bt.cpu()
        finally:
            ebv.set_debug(0)
    assert torch.equal(outs[0], outs[ebv.EBV_DEBUG_FORCE_EXACT])
    assert times[ebv.EBV_DEBUG_FORCE_EXACT] > times[0]


def test_flag_protocols_under_jitter(dev, ctx):
    """EBV_DEBUG_JITTER: random sleeps before every cross-CTA release of the
    wavefront solve and the vector path; results unchanged (bitwise), and the
    bounded waits never fire."""
    n = 1024
    d = ebv_inputs.generate(n, seed=12, nrhs=3, device=dev)
    A = d["At"].T
    ref = {}
    for flag in (0, ebv.EBV_DEBUG_JITTER):
        ebv.set_debug(flag, spin_timeout_s=20.0)
        try:
            ctx.set_path(ebv.EBV_PATH_VECTOR)
            LUv, _ = ebv.lu_factor(A, ctx=ctx)
            ctx.set_path(ebv.EBV_PATH_AUTO)
            LU, _ = ebv.lu_factor(A, ctx=ctx)
            X = ebv.lu_solve(LU, d["B"], ctx=ctx)
            torch.cuda.synchronize()
        finally:
            ebv.set_debug(0)
            ctx.set_path(ebv.EBV_PATH_AUTO)
        ref[flag] = (LUv.cpu(), LU.cpu(), X.cpu())
    for a, b in zip(ref[0], ref[ebv.EBV_DEBUG_JITTER]):
        assert torch.equal(a, b)
    lu_o, _ = oracle.lu_factor(A.cpu().numpy())
    assert bits_eq(ref[0][0].numpy(), lu_o)
    assert bits_eq(ref[0][2].numpy(), oracle.lu_solve(lu_o, d["B"].cpu().numpy()))


def test_set_debug_validation():
    assert ebv.ebv_set_debug(0, 0x80, 1.0) == 1
    assert ebv.ebv_set_debug(0, 0, -1.0) == 1
    assert ebv.ebv_set_debug(-1, 0, 1.0) == 1
