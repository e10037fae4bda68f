"""The C-ABI boundary without a GPU: libebv.so loads, exports every symbol
include/ebv.h declares, and its pure-host entry points (the EbV plan, the
block layouts, argument validation) agree bit-exactly with the oracle."""
import os
import re
import subprocess

import pytest

from oracle import ebv_plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ebv.h")


def _built_lib():
    from paper_1907_05767_b200 import _build
    return _build.build()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ebv_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("ebv_lu_factor", "ebv_lu_solve", "ebv_lu_factor_batched", "ebv_update"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _built_lib()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ebv_[a-z_0-9]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_binding_signatures_cover_the_header():
    import paper_1907_05767_b200 as ebv
    assert set(declared_symbols()) == set(ebv.SIGNATURES)
    L = ebv.lib()
    for name in ebv.SIGNATURES:
        assert getattr(L, name) is not None
        assert callable(getattr(ebv, name, None)), f"no Python binding named {name}"


def test_plan_units_match_oracle():
    import paper_1907_05767_b200 as ebv
    for n in list(range(2, 70)) + [128, 129, 511, 512]:
        for w in (1, 2, 3, 8):
            units, own = ebv.ebv_plan_units(n, w)
            ref = ebv_plan.equalize(ebv_plan.bivectorize(n), n)
            assert [tuple((t, k) for (t, k, _l) in u) for u in ref] == [tuple(u) for u in units]
            assert own == ebv_plan.assign(ref, w)


def test_owner_map_matches_oracle():
    import paper_1907_05767_b200 as ebv
    for n in (1, 2, 7, 8, 1023, 1024):
        for w in (1, 3, 128):
            assert ebv.ebv_plan_owner_map(n, w) == ebv_plan.column_pair_owner(n, w)


def test_block_owner_layouts():
    import paper_1907_05767_b200 as ebv
    N, P = 16, 4
    cyc = [ebv.ebv_block_owner(J, N, P, ebv.EBV_LAYOUT_CYCLIC) for J in range(N)]
    assert cyc == [J % P for J in range(N)]
    pair = [ebv.ebv_block_owner(J, N, P, ebv.EBV_LAYOUT_EBVPAIR) for J in range(N)]
    assert pair == ebv_plan.column_pair_owner(N, P)
    snake = [ebv.ebv_block_owner(J, N, P, ebv.EBV_LAYOUT_SNAKE) for J in range(N)]
    assert snake == [0, 1, 2, 3, 3, 2, 1, 0] * 2
    assert ebv.ebv_block_owner(N, N, P, ebv.EBV_LAYOUT_CYCLIC) == -1


def test_argument_validation_without_gpu():
    import paper_1907_05767_b200 as ebv
    L = ebv.lib()
    # NULL context is rejected synchronously (INVALID_VALUE = 1) before any CUDA call
    assert L.ebv_lu_factor(None, 4, None, 4, 0.0, None, None) == 1
    assert L.ebv_lu_solve(None, 4, None, 4, None, 4, 1, None) == 1
    assert L.ebv_update(None, 1, 1, 1, None, 1, None, 1, None, 1, None) == 1
    assert L.ebv_plan_owner_map(-1, 1, None) == 1
    assert L.ebv_block_width(None, 100) == 0
    assert L.ebv_lu_solve_batched(None, 4, None, 4, 16, 1, None, 4, 4, 1, None) == 1
    assert L.ebv_stats_timeline(None, None, 0) == -1
    assert L.ebv_normalize_unit_diagonal(None, 4, None, 4, None, 4, 1, None, None, None) == 1
    assert L.ebv_lu_to_ldu(None, 4, None, 4, None, None) == 1
    assert L.ebv_lu_factor_host(None, 4, None, 4, None, 4, 0.0, None, None) == 1
    assert L.ebv_lu_factor_banded(None, 4, 1, 1, None, 4, 0.0, None, None) == 1
    assert L.ebv_lu_solve_banded(None, 4, 1, 1, None, 4, None, 4, 1, None) == 1
    assert L.ebv_lu_factor_band(None, 4, 1, 1, None, 300, 0.0, None, None) == 1
    assert L.ebv_stream_wait_host_copy(None, None) == 1
    assert L.ebv_lu_solve_band(None, 4, 1, 1, None, 300, None, 4, 1, None) == 1
    assert ebv.batched_shard(10, 2, 3) == (7, 3) and ebv.batched_shard(0, 0, 4) == (0, 0)
    with pytest.raises(ebv.EbvError):
        ebv.batched_shard(10, 3, 3)
    assert ebv.ebv_status_string(0) == "success"
    assert ebv.ebv_status_string(5) == "not supported"


def test_no_cpu_fallback():
    """Without a CUDA device the tensor API refuses to run (no CPU path)."""
    import torch

    import paper_1907_05767_b200 as ebv
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(ebv.EbvError):
        ebv.Context(0)
