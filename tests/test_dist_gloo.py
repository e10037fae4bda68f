"""CPU, world_size 2 over gloo: the host logic of the multi-GPU path.

Each process takes the rank's column blocks from libebv's pure-host planner
(ebv_dist_local_blocks / ebv_block_owner), builds its slab, and runs the
step schedule of ebv_dist.cu — owner factors the panel, broadcast, every
rank substitutes / updates its blocks J > K — with numpy arithmetic and a
gloo broadcast in place of the GPU kernels and NCCL.  The assembled factors
must match the serial oracle (tolerance: numpy's summation order differs)
and the ranks' blocks must partition the matrix; the ring solve's protocol
(owner order, send / recv between consecutive owners, the final broadcast)
must give every rank the oracle's X.  This pins the planner, slab indexing,
panel packing and the broadcast / ring protocols on CPU."""
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


def _collect(procs, q, count, timeout=240):
    """count results from the queue; fails fast if a worker died."""
    import queue
    import time
    out, t0 = [], time.time()
    while len(out) < count:
        try:
            out.append(q.get(timeout=2))
        except queue.Empty:
            dead = [p.exitcode for p in procs if not p.is_alive() and p.exitcode not in (0, None)]
            assert not dead, f"worker failed: exit codes {dead}"
            assert time.time() - t0 < timeout, "timed out waiting for the workers"
    return out


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
        # ---- the ring solve of ebv_dist.cu (dist_solve): forward K ascending,
        # backward K descending; owner(K) receives the right-hand side from
        # the previous block's owner (when that is another rank), applies its
        # block column — diagonal block substituted, the rows below (forward)
        # or above (backward) updated — and sends it to the next block's
        # owner; X is broadcast from owner(0) at the end
        d = ebv_inputs.generate(n, seed=3, nrhs=2)
        b = d["B"].numpy().copy()
        for fwd in (True, False):
            order = range(N) if fwd else range(N - 1, -1, -1)
            for K in order:
                own = ebv.ebv_block_owner(K, N, world, layout)
                prev, nxt = (K - 1, K + 1) if fwd else (K + 1, K - 1)
                if own != rank:
                    continue
                bt = torch.from_numpy(b)
                if 0 <= prev < N and ebv.ebv_block_owner(prev, N, world, layout) != rank:
                    dist.recv(bt, src=ebv.ebv_block_owner(prev, N, world, layout))
                b = bt.numpy()
                c0, w = K * nb, min(nb, n - K * nb)
                col = slab[:, loc[K]:loc[K] + w]
                if fwd:
                    L11 = np.tril(col[c0:c0 + w], -1) + np.eye(w)
                    b[c0:c0 + w] = np.linalg.solve(L11, b[c0:c0 + w])
                    b[c0 + w:] -= col[c0 + w:] @ b[c0:c0 + w]
                else:
                    U11 = np.triu(col[c0:c0 + w])
                    b[c0:c0 + w] = np.linalg.solve(U11, b[c0:c0 + w])
                    b[:c0] -= col[:c0] @ b[c0:c0 + w]
                if 0 <= nxt < N and ebv.ebv_block_owner(nxt, N, world, layout) != rank:
                    dist.send(torch.from_numpy(np.ascontiguousarray(b)),
                              dst=ebv.ebv_block_owner(nxt, N, world, layout))
        bt = torch.from_numpy(np.ascontiguousarray(b))
        dist.broadcast(bt, src=ebv.ebv_block_owner(0, N, world, layout))
        x_ring = bt.numpy().copy()
        out = torch.from_numpy(np.ascontiguousarray(slab.T))
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, cols, out, x_ring))
        if rank == 0:   # plain numpy through the queue (no shared-memory tensors)
            gathered = [(r, c, o.numpy().copy(), x) for r, c, o, x in gathered]
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
    res = _collect(procs, q, world)
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
    for _, cols, out, _x in gathered:
        full[:, cols] = out.T
    import ebv_inputs
    d = ebv_inputs.generate(n, seed=3, nrhs=2)
    A = d["At"].T.numpy()
    lu_o, _ = oracle.lu_factor(A)
    assert np.max(np.abs(full - lu_o)) <= 1e-12 * np.max(np.abs(lu_o))
    # the ring solve: every rank ends with the same X, equal to the oracle's
    # solve (tolerance: numpy's order) and to the exact solution
    x_o = oracle.lu_solve(lu_o, d["B"].numpy())
    xs = [x for _, _, _, x in gathered]
    assert all(np.array_equal(xs[0], x) for x in xs)
    assert np.max(np.abs(xs[0] - x_o)) <= 1e-12 * np.max(np.abs(x_o))
    assert np.max(np.abs(xs[0] - d["X"].numpy())) <= 1e-10


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
    gathered = _collect(procs, q, 1)[0]
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
