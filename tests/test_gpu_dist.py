"""GPU: the 1D block-cyclic multi-GPU schedule.

On one B200 the P-rank schedule runs in emulation (all virtual ranks' slabs
in one process) and, for P = 1, through a real NCCL communicator.  Every
result is compared BITWISE with the serial oracle and with the one-GPU
blocked schedule of the same block width (the per-entry order does not
depend on P)."""
import numpy as np
import pytest
import torch

import ebv_inputs
import oracle

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


def slabs_for(d, n, nb, P, layout, dev):
    """Per-rank column-major slabs (storage (cols, n): row c = column c)."""
    slabs, colmaps = [], []
    for r in range(P):
        cols = ebv.dist_local_columns(n, nb, r, P, layout)
        st = d["At"][torch.tensor(cols, dtype=torch.long, device=dev)].clone() if cols else \
            torch.zeros(1, n, dtype=torch.float64, device=dev)
        slabs.append(st)
        colmaps.append(cols)
    return slabs, colmaps


def assemble(slabs, colmaps, n):
    full = np.zeros((n, n))
    for st, cols in zip(slabs, colmaps):
        if cols:
            full[:, cols] = st[: len(cols)].T.cpu().numpy()
    return full


@pytest.mark.parametrize("P,nb,layout,n", [(1, 128, 0, 700), (2, 64, 0, 1000), (3, 128, 0, 1000), (4, 64, 1, 1537),
                                           (8, 64, 2, 1000), (4, 256, 0, 2100), (2, 128, 1, 64), (8, 64, 0, 300)])
def test_emulated_dist_factor_and_solve_bitwise(dev, ctx, P, nb, layout, n):
    d = ebv_inputs.generate(n, seed=P * 1000 + nb + layout, nrhs=2, device=dev)
    slabs, colmaps = slabs_for(d, n, nb, P, layout, dev)
    info = torch.zeros((), dtype=torch.int64, device=dev)
    sh = torch.cuda.current_stream().cuda_stream
    st = ebv.ebv_lu_factor_dist_emulated(ctx.handle, n, P, nb, layout, [s.data_ptr() for s in slabs], n, 0.0,
                                         info.data_ptr(), sh)
    assert st == 0, ebv.ebv_last_error()
    B = d["B"].T.clone(memory_format=torch.contiguous_format)   # (nrhs, n) = column-major n x nrhs
    st = ebv.ebv_lu_solve_dist_emulated(ctx.handle, n, P, nb, layout, [s.data_ptr() for s in slabs], n,
                                        B.data_ptr(), n, 2, sh)
    assert st == 0, ebv.ebv_last_error()
    torch.cuda.synchronize()
    lu_g = assemble(slabs, colmaps, n)
    lu_o, info_o = oracle.lu_factor(d["At"].T.cpu().numpy())
    assert int(info) == info_o == 0
    assert bits_eq(lu_g, lu_o)
    x_o = oracle.lu_solve(lu_o, d["B"].cpu().numpy())
    assert bits_eq(B.T.cpu().numpy(), x_o)
    # the one-GPU blocked schedule with the same block width is the same computation
    ctx.set_block(nb)
    LU1, _ = ebv.lu_factor(d["At"].T, ctx=ctx)
    ctx.set_block(0)
    torch.cuda.synchronize()
    assert bits_eq(LU1.cpu().numpy(), lu_g)


@pytest.mark.parametrize("P,nb,n,nrhs", [(3, 64, 700, 20), (2, 128, 1000, 16), (5, 64, 333, 3)])
def test_emulated_dist_solve_many_rhs_bitwise(dev, ctx, P, nb, n, nrhs):
    """The ring solve in right-hand-side groups of 16 (and a ragged last
    block): bitwise the oracle."""
    d = ebv_inputs.generate(n, seed=n + nrhs, nrhs=nrhs, device=dev)
    slabs, colmaps = slabs_for(d, n, nb, P, 0, dev)
    info = torch.zeros((), dtype=torch.int64, device=dev)
    sh = torch.cuda.current_stream().cuda_stream
    assert ebv.ebv_lu_factor_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n, 0.0,
                                           info.data_ptr(), sh) == 0, ebv.ebv_last_error()
    B = d["B"].T.clone(memory_format=torch.contiguous_format)
    for _ in range(2):   # twice: the flags' epochs advance per call
        Bw = B.clone()
        assert ebv.ebv_lu_solve_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n,
                                              Bw.data_ptr(), n, nrhs, sh) == 0, ebv.ebv_last_error()
        torch.cuda.synchronize()
        lu_o, _ = oracle.lu_factor(d["At"].T.cpu().numpy())
        assert bits_eq(Bw.T.cpu().numpy(), oracle.lu_solve(lu_o, d["B"].cpu().numpy()))


def test_emulated_dist_info(dev, ctx):
    n, nb, P = 400, 64, 3
    A = torch.eye(n, dtype=torch.float64, device=dev) * 3.0
    A[200, 200] = 0.0
    A[350, 350] = 0.0
    d = {"At": A.T.contiguous()}
    slabs, _ = slabs_for(d, n, nb, P, 0, dev)
    info = torch.zeros((), dtype=torch.int64, device=dev)
    st = ebv.ebv_lu_factor_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n, 0.0,
                                         info.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    assert int(info) == 201


def test_real_nccl_single_rank(dev):
    """ebv_create_dist + ebv_lu_factor_dist / ebv_lu_solve_dist through a real
    NCCL communicator (1 rank on this GPU)."""
    n, nb = 900, 128
    uid = ebv.ebv_get_unique_id()
    h = ebv.ebv_create_dist(0, uid, 0, 1, nb, 0)
    try:
        d = ebv_inputs.generate(n, seed=77, nrhs=1, device=dev)
        slab = d["At"].clone()
        info = torch.zeros((), dtype=torch.int64, device=dev)
        sh = torch.cuda.current_stream().cuda_stream
        assert ebv.ebv_lu_factor_dist(h, n, slab.data_ptr(), n, 0.0, info.data_ptr(), sh) == 0, ebv.ebv_last_error()
        B = d["B"].T.clone(memory_format=torch.contiguous_format)
        assert ebv.ebv_lu_solve_dist(h, n, slab.data_ptr(), n, B.data_ptr(), n, 1, sh) == 0, ebv.ebv_last_error()
        torch.cuda.synchronize()
        lu_o, _ = oracle.lu_factor(d["At"].T.cpu().numpy())
        assert bits_eq(slab.T.cpu().numpy(), lu_o)
        assert bits_eq(B.T.cpu().numpy(), oracle.lu_solve(lu_o, d["B"].cpu().numpy()))
        assert int(info) == 0
    finally:
        ebv.ebv_destroy(h)


def test_dist_errors(dev, ctx):
    L = ebv.lib()
    info = torch.zeros((), dtype=torch.int64, device=dev)
    # not a distributed context
    assert L.ebv_lu_factor_dist(ctx.handle, 4, None, 4, 0.0, info.data_ptr(), None) == 1
    # a distributed context is rejected by the single-GPU entry points
    uid = ebv.ebv_get_unique_id()
    h = ebv.ebv_create_dist(0, uid, 0, 1, 64, 0)
    try:
        A = torch.eye(4, dtype=torch.float64, device=dev)
        assert L.ebv_lu_factor(h, 4, A.data_ptr(), 4, 0.0, info.data_ptr(), None) == 1
        assert L.ebv_lu_solve(h, 4, A.data_ptr(), 4, A.data_ptr(), 4, 1, None) == 1
        assert L.ebv_lu_factor_host(h, 4, A.cpu().data_ptr(), 4, A.data_ptr(), 4, 0.0, info.data_ptr(), None) == 1
    finally:
        ebv.ebv_destroy(h)


@pytest.mark.parametrize("P,nb,n", [(3, 64, 700), (2, 128, 1000), (1, 64, 300)])
def test_emulated_dist_default_pivot_floor(dev, ctx, P, nb, n):
    """tau < 0 in the distributed schedule: the default floor n*eps*||A||_inf
    from the ranks' partial row sums (added in rank order here, by an NCCL
    all-reduce on real ranks) — the same floor and the same info as the
    single-GPU factorization (the generator's row sums are exact)."""
    d = ebv_inputs.generate(n, seed=n + P, nrhs=1, device=dev)
    At = d["At"].clone()
    k = 2 * nb + 5
    At[:, k] = 0.0             # row k and column k of A zero: an isolated 1 x 1 block,
    At[k, :] = 0.0             # so u_kk = a_kk = 1e-300, far below the default floor
    At[k, k] = 1e-300          # (info = k + 1), and every other factor entry stays finite
    slabs, colmaps = slabs_for({"At": At}, n, nb, P, 0, dev)
    info = torch.zeros((), dtype=torch.int64, device=dev)
    sh = torch.cuda.current_stream().cuda_stream
    assert ebv.ebv_lu_factor_dist_emulated(ctx.handle, n, P, nb, 0, [s.data_ptr() for s in slabs], n, -1.0,
                                           info.data_ptr(), sh) == 0, ebv.ebv_last_error()
    ctx.set_block(nb)
    LU1, info1 = ebv.lu_factor(At.T, tau=-1.0, ctx=ctx)
    ctx.set_block(0)
    torch.cuda.synchronize()
    assert int(info) == int(info1) > 0
    assert bits_eq(assemble(slabs, colmaps, n), LU1.cpu().numpy())


_FORCED_SNIPPET = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, ebv_inputs, oracle
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
ebv.load_nccl()
for n, nb, tau in ((900, 128, -1.0), (1536, 256, 0.0)):
    uid = ebv.ebv_get_unique_id()
    h = ebv.ebv_create_dist(0, uid, 0, 1, nb, 0)
    d = ebv_inputs.generate(n, seed=5 + n, nrhs=2, device=dev)
    lu_o, info_o = oracle.lu_factor(d["At"].T.cpu().numpy())
    x_o = oracle.lu_solve(lu_o, d["B"].cpu().numpy())
    slab = torch.empty_like(d["At"])
    info = torch.zeros((), dtype=torch.int64, device=dev)
    s = torch.cuda.Stream(dev)   # a created stream: the second call captures a graph, later calls replay it
    sh = s.cuda_stream
    for rep in range(4):
        with torch.cuda.stream(s):
            slab.copy_(d["At"])
            assert ebv.ebv_lu_factor_dist(h, n, slab.data_ptr(), n, tau, info.data_ptr(), sh) == 0, ebv.ebv_last_error()
            B = d["B"].T.clone(memory_format=torch.contiguous_format)
            assert ebv.ebv_lu_solve_dist(h, n, slab.data_ptr(), n, B.data_ptr(), n, 2, sh) == 0, ebv.ebv_last_error()
        torch.cuda.synchronize()
        assert np.array_equal(slab.T.cpu().numpy().view(np.uint64), lu_o.view(np.uint64)), rep
        assert np.array_equal(B.T.cpu().numpy().view(np.uint64), x_o.view(np.uint64)), rep
        assert int(info) == info_o == 0
    ebv.ebv_destroy(h)
print("forced NCCL data path bitwise ok")
"""


def test_real_nccl_single_rank_data_path():
    """The NCCL data path itself on one GPU: with EBV_DIST_FORCE_NCCL=1 a
    one-rank communicator still broadcasts every panel, all-reduces info and
    (tau < 0) the row sums, and runs the ring solve with its final
    broadcast — a one-rank collective is a local copy, so the calls, streams
    and event protocol of the multi-rank schedule execute and must leave the
    results bitwise the oracle's, also when the schedule is captured into a
    CUDA graph (second call) and replayed (later calls).  (The switch is read
    once per process.)"""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EBV_DIST_FORCE_NCCL="1")
    r = subprocess.run([sys.executable, "-c", _FORCED_SNIPPET, root], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bitwise ok" in r.stdout
