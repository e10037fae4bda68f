"""EbV plan oracle (paper Eq 7) and the shared input generator."""
import numpy as np
import pytest
import torch

import ebv_inputs
from oracle import ebv_plan


def test_plan_golden(golden):
    for ex in golden["plan"]:
        n = ex["n"]
        d = ebv_plan.bivectorize(n)
        if "lengths_L" in ex:
            assert [x[2] for x in d if x[0] == "L"] == ex["lengths_L"], ex["cite"]
            assert [x[2] for x in d if x[0] == "U"] == ex["lengths_U"], ex["cite"]
        if "units" in ex:
            units = ebv_plan.equalize(d, n)
            got = [[[t, k] for (t, k, _l) in u] for u in units]
            assert got == ex["units"], ex["cite"]
    for ex in golden["assign"]:
        n, w = ex["n"], ex["workers"]
        units = ebv_plan.equalize(ebv_plan.bivectorize(n), n)
        own = ebv_plan.assign(units, w)
        if "owners" in ex:
            assert own == ex["owners"], ex["cite"]
        lengths, counts = ebv_plan.plan_stats(units, own, w)
        if "lengths" in ex:
            assert lengths == ex["lengths"], ex["cite"]
        if "unit_counts" in ex:
            assert counts == ex["unit_counts"], ex["cite"]


def test_plan_invariants_all_n():
    """(n-1) units in total, all of equal length n."""
    for n in range(2, 513):
        units = ebv_plan.equalize(ebv_plan.bivectorize(n), n)
        assert len(units) == n - 1
        assert all(sum(d[2] for d in u) == n for u in units)
        for w in (1, 2, 3, 7, 8):
            if w > n - 1:
                continue
            lengths, counts = ebv_plan.plan_stats(units, ebv_plan.assign(units, w), w)
            assert max(lengths) - min(lengths) <= n
            assert max(counts) - min(counts) <= 1


def test_plan_disjoint_cover():
    for n in range(2, 65):
        units = ebv_plan.equalize(ebv_plan.bivectorize(n), n)
        pos = [p for u in units for p in ebv_plan.unit_positions(u, n)]
        want = [(i, j) for i in range(n) for j in range(n) if i != j]
        assert sorted(pos) == sorted(want)


def test_column_pair_owner_balance():
    """Paired indices (j, n-1-j) share an owner; lengths of the paired columns'
    on-or-below-diagonal parts sum to n+1 for every pair."""
    for n in (8, 9, 1024):
        own = ebv_plan.column_pair_owner(n, 4)
        for j in range(n):
            assert own[j] == own[n - 1 - j]
            assert (n - j) + (n - (n - 1 - j)) == n + 1


# ---------------------------------------------------------------- generator
def test_generator_dominance_and_exact_b():
    d = ebv_inputs.generate(300, seed=5, nrhs=3)
    a = d["At"].T.numpy()
    off = np.abs(a).sum(1) - np.abs(np.diag(a))
    assert np.all(np.abs(np.diag(a)) - off == 1.0)        # margin exactly 1
    assert np.all(np.abs(a - np.diag(np.diag(a))) < 1.0)
    # on the 2^-30 grid
    assert np.all(a * 2.0 ** 30 == np.round(a * 2.0 ** 30))
    # B = A X exactly: integer arithmetic in units of 2^-30
    au = (a * 2.0 ** 30).astype(np.int64)
    xu = d["X"].numpy().astype(np.int64)
    assert np.array_equal((au @ xu).astype(np.float64) * 2.0 ** -30, d["B"].numpy())
    assert set(np.unique(xu)) <= set(range(-4, 5))


def test_generator_determinism_and_slab():
    d1 = ebv_inputs.generate(200, seed=9)
    d2 = ebv_inputs.generate(200, seed=9, chunk=37)
    assert torch.equal(d1["At"], d2["At"]) and torch.equal(d1["B"], d2["B"])
    cols = torch.tensor([3, 4, 100, 199])
    d3 = ebv_inputs.generate(200, seed=9, cols=cols)
    assert torch.equal(d3["At"], d1["At"][cols])
    assert not torch.equal(ebv_inputs.generate(200, seed=10)["At"], d1["At"])


def test_batched_generator_matches_dense_generator():
    db = ebv_inputs.generate_batched(4, 32, seed=2, nrhs=1, first_system=10)
    for s in range(4):
        d = ebv_inputs.generate(32, seed=2, system=10 + s)
        assert torch.equal(db["At"][s], d["At"])
        assert torch.equal(db["B"][s], d["B"])


def test_hash_known_values():
    """lowbias32 reference values (computed by hand-checked uint32 arithmetic)."""
    def ref(x):
        M = 0xFFFFFFFF
        x ^= x >> 16
        x = (x * 0x7FEB352D) & M
        x ^= x >> 15
        x = (x * 0x846CA68B) & M
        x ^= x >> 16
        return x
    xs = [0, 1, 2, 12345, 0xFFFFFFFF, 0x80000000]
    got = ebv_inputs.hash32(torch.tensor(xs, dtype=torch.int64)).tolist()
    assert got == [ref(x) for x in xs]
