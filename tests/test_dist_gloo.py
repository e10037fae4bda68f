"""CPU, world_size 2 over gloo: the host logic of the multi-GPU path.

Each process takes the rank's column blocks from libebv's pure-host planner
(ebv_dist_local_blocks / ebv_block_owner), builds its slab, and runs the
step schedule of ebv_dist.cu — owner factors the panel, broadcast, every
rank substitutes / updates its blocks J > K — with numpy arithmetic and a
gloo broadcast in place of the GPU kernels and NCCL.  The assembled factors
must match the serial oracle (tolerance: numpy's summation order differs)
and the ranks' blocks must partition the matrix.  This pins the planner,
slab indexing, panel packing and the broadcast protocol on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _panel_lu(P, w):
    """In-place LU of a tall panel (M x w): Eq 6 restricted to w steps."""
    for k in range(w):
        P[k + 1:, k] /= P[k, k]
        P[k + 1:, k + 1:w] -= np.outer(P[k + 1:, k], P[k, k + 1:w])


def _worker(rank, world, port, n, nb, layout, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ebv_inputs
        import paper_1907_05767_b200 as ebv
        blocks, cols_w = ebv.ebv_dist_local_blocks(n, nb, rank, world, layout)
        cols = ebv.dist_local_columns(n, nb, rank, world, layout)
        assert len(cols) == cols_w
        A = ebv_inputs.generate(n, seed=3)["At"].T.numpy()
        slab = np.array(A[:, cols], order="F")            # n x local_cols
        loc = {J: i * 0 for i, J in enumerate(blocks)}
        off = 0
        for J in blocks:
            loc[J] = off
            off += min(nb, n - J * nb)
        N = (n + nb - 1) // nb
        for K in range(N):
            c0, w = K * nb, min(nb, n - K * nb)
            M = n - c0
            owner = ebv.ebv_block_owner(K, N, world, layout)
            pbuf = torch.zeros(M * w, dtype=torch.float64)
            if owner == rank:
                P = slab[c0:, loc[K]:loc[K] + w]
                _panel_lu(P, w)
                pbuf[:] = torch.from_numpy(np.asfortranarray(P).ravel(order="F"))
            dist.broadcast(pbuf, src=owner)
            panel = pbuf.numpy().reshape((M, w), order="F")
            rest = [i for i, J in enumerate(blocks) if J > K]
            if rest:
                lc0 = loc[blocks[rest[0]]]
                X = slab[c0:c0 + w, lc0:]
                L11 = np.tril(panel[:w, :w], -1) + np.eye(w)
                X[:] = np.linalg.solve(L11, X)            # U12 = L11^-1 A12
                slab[c0 + w:, lc0:] -= panel[w:, :] @ X   # A22 -= L21 U12
        out = torch.from_numpy(np.ascontiguousarray(slab.T))
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, cols, out))
        if rank == 0:   # plain numpy through the queue (no shared-memory tensors)
            gathered = [(r, c, o.numpy().copy()) for r, c, o in gathered]
        q.put((rank, blocks, gathered if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,nb,layout", [(300, 64, 0), (257, 64, 1), (200, 64, 2)])
def test_gloo_world2_block_cyclic_schedule(n, nb, layout):
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, nb, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    # the ranks' blocks partition all column blocks
    N = (n + nb - 1) // nb
    all_blocks = sorted(b for _, blocks, _ in res for b in blocks)
    assert all_blocks == list(range(N))
    gathered = res[0][2]
    full = np.zeros((n, n))
    for _, cols, out in gathered:
        full[:, cols] = out.T
    import ebv_inputs
    A = ebv_inputs.generate(n, seed=3)["At"].T.numpy()
    lu_o, _ = oracle.lu_factor(A)
    assert np.max(np.abs(full - lu_o)) <= 1e-12 * np.max(np.abs(lu_o))


def _batched_worker(rank, world, port, batch, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ebv_inputs
        import oracle
        import paper_1907_05767_b200 as ebv
        first, count = ebv.batched_shard(batch, rank, world)
        d = ebv_inputs.generate_batched(count, n, seed=5, nrhs=1, first_system=first)
        lu, x, info = oracle.lu_factor_batched(d["At"].transpose(1, 2).numpy(), d["B"].numpy())
        # no collective on the data path; results gathered only to check them
        gathered = [None] * world
        dist.all_gather_object(gathered, (first, count, x))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch,n", [(7, 32), (10, 5)])
def test_gloo_world2_batched_sharding(batch, n):
    """C5 sharding: each rank takes ebv_batched_shard's
    contiguous range, generates its systems (generator offset by the first
    system index) and solves them alone; the union equals the unsharded
    computation bitwise and the ranges partition the batch."""
    import ebv_inputs
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batched_worker, args=(r, world, port, batch, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    firsts = sorted((f, c) for f, c, _ in gathered)
    assert firsts[0][0] == 0 and sum(c for _, c in firsts) == batch
    assert all(firsts[i][0] + firsts[i][1] == firsts[i + 1][0] for i in range(len(firsts) - 1))
    full = ebv_inputs.generate_batched(batch, n, seed=5, nrhs=1)
    _, x_full, _ = oracle.lu_factor_batched(full["At"].transpose(1, 2).numpy(), full["B"].numpy())
    x_sh = np.concatenate([x for f, c, x in sorted(gathered, key=lambda g: g[0])])
    assert np.array_equal(x_sh.view(np.uint64), x_full.view(np.uint64))
