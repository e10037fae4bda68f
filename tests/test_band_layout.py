"""Compact band storage (include/ebv.h, ebv_lu_factor_band): the layout
helpers and the band generator are pinned against the dense generator —
generate_band must give generate(kl, ku)'s entries bit for bit, and
band_pack / band_unpack must be exact inverses on banded matrices.  CPU only
(layout, no arithmetic of the method)."""
import torch

import ebv_inputs
import paper_1907_05767_b200 as ebv


def test_generate_band_equals_dense_generator():
    for n, kl, ku, seed in ((1, 0, 0, 1), (40, 3, 7, 2), (300, 17, 29, 5), (257, 256, 1, 9)):
        d = ebv_inputs.generate(n, seed=seed, kl=kl, ku=ku)
        ld = ebv.band_ld(kl, ku)
        g = ebv_inputs.generate_band(n, kl, ku, ebv.EBV_BAND_PAD, ld, seed=seed)
        A = d["At"].T
        assert torch.equal(ebv.band_pack(A, kl, ku), g["AB"])
        assert torch.equal(d["B"], g["B"]) and torch.equal(d["X"], g["X"])
        assert torch.equal(ebv.band_unpack(g["AB"], n, kl, ku), A)


def test_band_storage_layout():
    n, kl, ku = 50, 4, 6
    ld = ebv.band_ld(kl, ku)
    assert ld % 2 == 1 and ld >= kl + ku + 2 * ebv.EBV_BAND_PAD + 1
    A = torch.zeros(n, n, dtype=torch.float64)
    for i in range(n):
        for j in range(max(0, i - kl), min(n, i + ku + 1)):
            A[i, j] = 1000 * i + j + 1
    AB = ebv.band_pack(A, kl, ku)
    flat = AB.reshape(-1)          # column-major ldab x n storage
    for i, j in ((0, 0), (3, 0), (0, 6), (49, 49), (45, 49), (49, 45)):
        assert flat[(ebv.EBV_BAND_PAD + ku + i - j) + j * ld] == A[i, j]
    # everything outside the band slots is zero
    mask = torch.zeros_like(AB, dtype=torch.bool)
    for d in range(-ku, kl + 1):
        mask[:, ebv.EBV_BAND_PAD + ku + d] = True
    assert (AB[~mask] == 0).all()
