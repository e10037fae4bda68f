"""paper_1907_05767_b200 — B200 (sm_100a) implementation of the hot path of the
"Equal bi-Vectorized" (EbV) method (arXiv 1907.05767): no-pivot LU factor
A = LU of diagonally dominant fp64 matrices followed by forward (LY = B) and
backward (UX = Y) substitution (Eq 1, Eq 6 of the paper).

This module is a thin binding over the C ABI of ``libebv.so``
(include/ebv.h): argument marshalling only — every step of the path runs in
the library's CUDA kernels.  PyTorch is used for device memory and streams.
There is no CPU fallback: if the library is missing, every call raises.

Two layers:
  * the C-ABI mirror, same names as include/ebv.h (``ebv_lu_factor(ctx, n,
    A_ptr, lda, tau, info_ptr, stream)`` ...), taking raw device pointers;
  * tensor helpers (``lu_factor``, ``lu_solve``, ``lu_factor_batched``,
    ``Context``) that take torch CUDA float64 tensors in logical [i, j]
    indexing and pass column-major storage to the library.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libebv.so")

EBV_SUCCESS = 0
EBV_PATH_AUTO, EBV_PATH_VECTOR, EBV_PATH_BLOCKED, EBV_PATH_LEFT = 0, 1, 2, 3
EBV_LAYOUT_CYCLIC, EBV_LAYOUT_EBVPAIR, EBV_LAYOUT_SNAKE = 0, 1, 2
EBV_BAND_PAD = 128   # include/ebv.h: padding rows above and below the band in compact band storage
KCLASSES = ["gemm_dmma", "leaf_lu", "trsm", "solve", "batched", "vector", "other", "update"]

# every exported symbol of include/ebv.h with its ctypes signature
_i64, _i32, _vp, _d, _int = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double, ctypes.c_int
SIGNATURES = {
    "ebv_create": (_int, [ctypes.POINTER(_vp), _int]),
    "ebv_destroy": (_int, [_vp]),
    "ebv_status_string": (ctypes.c_char_p, [_int]),
    "ebv_last_error": (ctypes.c_char_p, []),
    "ebv_set_path": (_int, [_vp, _int]),
    "ebv_set_leaf": (_int, [_vp, _i64]),
    "ebv_set_vector_ctas": (_int, [_vp, _i64]),
    "ebv_set_block": (_int, [_vp, _i64]),
    "ebv_block_width": (_i64, [_vp, _i64]),
    "ebv_lu_factor_banded": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _d, _vp, _vp]),
    "ebv_lu_solve_banded": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "ebv_lu_factor_band": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _d, _vp, _vp]),
    "ebv_stream_wait_host_copy": (_int, [_vp, _vp]),
    "ebv_lu_solve_band": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "ebv_batched_shard": (_int, [_i64, _int, _int, _vp, _vp]),
    "ebv_lu_factor_host": (_int, [_vp, _i64, _vp, _i64, _vp, _i64, _d, _vp, _vp]),
    "ebv_stats_timeline": (_i64, [_vp, _vp, _i64]),
    "ebv_set_lookahead": (_int, [_vp, _int]),
    "ebv_set_graphs": (_int, [_vp, _int]),
    "ebv_lu_factor": (_int, [_vp, _i64, _vp, _i64, _d, _vp, _vp]),
    "ebv_lu_solve": (_int, [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "ebv_lu_factor_batched": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _d, _vp, _vp]),
    "ebv_lu_solve_batched": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _vp]),
    "ebv_normalize_unit_diagonal": (_int, [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ebv_lu_to_ldu": (_int, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "ebv_update": (_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "ebv_get_unique_id": (_int, [_vp]),
    "ebv_create_dist": (_int, [ctypes.POINTER(_vp), _int, _vp, _int, _int, _i64, _int]),
    "ebv_dist_local_blocks": (_int, [_i64, _i64, _int, _int, _int, _vp, _i64, ctypes.POINTER(_i64),
                                     ctypes.POINTER(_i64)]),
    "ebv_lu_factor_dist": (_int, [_vp, _i64, _vp, _i64, _d, _vp, _vp]),
    "ebv_lu_solve_dist": (_int, [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp]),
    "ebv_lu_factor_dist_emulated": (_int, [_vp, _i64, _int, _i64, _int, _vp, _i64, _d, _vp, _vp]),
    "ebv_lu_solve_dist_emulated": (_int, [_vp, _i64, _int, _i64, _int, _vp, _i64, _vp, _i64, _i64, _vp]),
    "ebv_plan_owner_map": (_int, [_i64, _i64, _vp]),
    "ebv_plan_units": (_int, [_i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "ebv_block_owner": (_i64, [_i64, _i64, _i64, _int]),
    "ebv_stats_enable": (_int, [_vp, _int]),
    "ebv_stats_reset": (_int, [_vp]),
    "ebv_stats_get": (_int, [_vp, _int, ctypes.POINTER(_i64), ctypes.POINTER(_d), ctypes.POINTER(_d),
                             ctypes.POINTER(_d)]),
    "ebv_launch_count": (_i64, [_vp]),
    "ebv_set_debug": (_int, [_int, ctypes.c_uint, _d]),
    "ebv_dist_nranks": (_int, [_vp]),
}
EBV_DEBUG_FORCE_EXACT, EBV_DEBUG_JITTER = 1, 2

_lib = None


class EbvError(RuntimeError):
    pass


def lib():
    """Load libebv.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EbvError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != EBV_SUCCESS:
        L = lib()
        raise EbvError(f"{what}: {L.ebv_status_string(status).decode()} ({L.ebv_last_error().decode()})")


# ------------------------------------------------------------------ C-ABI mirror
def ebv_create(device: int = 0) -> int:
    h = _vp()
    _check(lib().ebv_create(ctypes.byref(h), device), "ebv_create")
    return h.value


def ebv_destroy(ctx: int) -> int:
    return lib().ebv_destroy(ctx)


def ebv_status_string(s: int) -> str:
    return lib().ebv_status_string(s).decode()


def ebv_last_error() -> str:
    return lib().ebv_last_error().decode()


def ebv_set_path(ctx, path):
    return lib().ebv_set_path(ctx, path)


def ebv_set_leaf(ctx, leaf):
    return lib().ebv_set_leaf(ctx, leaf)


def ebv_set_block(ctx, nb):
    return lib().ebv_set_block(ctx, nb)


def ebv_block_width(ctx, n):
    return lib().ebv_block_width(ctx, n)


def ebv_set_lookahead(ctx, enable):
    return lib().ebv_set_lookahead(ctx, 1 if enable else 0)


def ebv_set_graphs(ctx, enable):
    return lib().ebv_set_graphs(ctx, 1 if enable else 0)


def ebv_set_vector_ctas(ctx, ctas):
    return lib().ebv_set_vector_ctas(ctx, ctas)


def ebv_lu_factor(ctx, n, A, lda, tau, d_info, stream):
    return lib().ebv_lu_factor(ctx, n, A, lda, tau, d_info, stream)


def ebv_lu_solve(ctx, n, LU, lda, B, ldb, nrhs, stream):
    return lib().ebv_lu_solve(ctx, n, LU, lda, B, ldb, nrhs, stream)


def ebv_lu_factor_batched(ctx, n, A, lda, strideA, batch, B, ldb, strideB, nrhs, tau, d_info, stream):
    return lib().ebv_lu_factor_batched(ctx, n, A, lda, strideA, batch, B, ldb, strideB, nrhs, tau, d_info, stream)


def ebv_lu_solve_batched(ctx, n, LU, lda, strideA, batch, B, ldb, strideB, nrhs, stream):
    return lib().ebv_lu_solve_batched(ctx, n, LU, lda, strideA, batch, B, ldb, strideB, nrhs, stream)


def ebv_batched_shard(batch, rank, nranks, first, count):
    return lib().ebv_batched_shard(batch, rank, nranks, first, count)


def batched_shard(batch: int, rank: int, nranks: int):
    """(first, count) of rank's contiguous share of `batch` systems (C5 sharding)."""
    f, c = ctypes.c_int64(), ctypes.c_int64()
    _check(ebv_batched_shard(batch, rank, nranks, ctypes.byref(f), ctypes.byref(c)), "ebv_batched_shard")
    return f.value, c.value


def ebv_lu_factor_banded(ctx, n, kl, ku, A, lda, tau, d_info, stream):
    return lib().ebv_lu_factor_banded(ctx, n, kl, ku, A, lda, tau, d_info, stream)


def ebv_lu_solve_banded(ctx, n, kl, ku, LU, lda, B, ldb, nrhs, stream):
    return lib().ebv_lu_solve_banded(ctx, n, kl, ku, LU, lda, B, ldb, nrhs, stream)


def lu_factor_banded(A: torch.Tensor, kl: int, ku: int, tau: float = 0.0, ctx: Context | None = None):
    """Zero-skip LU of a banded A (entries outside the band must be zero):
    returns (LU, info) like lu_factor."""
    _require(A, "A")
    n = A.shape[0]
    ctx = ctx or default_context(A.device.index or 0)
    LU = A.mT.contiguous().mT.clone() if _colmajor_ld(A) < 0 else A.clone()
    info = torch.zeros((), dtype=torch.int64, device=A.device)
    _check(ebv_lu_factor_banded(ctx.handle, n, kl, ku, LU.data_ptr(), max(_colmajor_ld(LU), 1), float(tau),
                                info.data_ptr(), _stream_handle(A.device)), "ebv_lu_factor_banded")
    return LU, info


def lu_solve_banded(LU: torch.Tensor, B: torch.Tensor, kl: int, ku: int, ctx: Context | None = None):
    """X from the banded factors (zero tiles skipped); B (n,) or (n, nrhs)."""
    _require(LU, "LU")
    n = LU.shape[0]
    ctx = ctx or default_context(LU.device.index or 0)
    vec = B.dim() == 1
    X = B.reshape(n, -1).mT.contiguous().mT.clone()
    _check(ebv_lu_solve_banded(ctx.handle, n, kl, ku, LU.data_ptr(), max(_colmajor_ld(LU), 1), X.data_ptr(),
                               max(n, 1), X.shape[1], _stream_handle(LU.device)), "ebv_lu_solve_banded")
    return X[:, 0] if vec else X


def ebv_stream_wait_host_copy(ctx, stream):
    return lib().ebv_stream_wait_host_copy(ctx, stream)


def ebv_lu_factor_band(ctx, n, kl, ku, AB, ldab, tau, d_info, stream):
    return lib().ebv_lu_factor_band(ctx, n, kl, ku, AB, ldab, tau, d_info, stream)


def ebv_lu_solve_band(ctx, n, kl, ku, AB, ldab, B, ldb, nrhs, stream):
    return lib().ebv_lu_solve_band(ctx, n, kl, ku, AB, ldab, B, ldb, nrhs, stream)


def band_ld(kl: int, ku: int) -> int:
    """Smallest leading dimension of compact band storage (odd, so the dense
    view's leading dimension ldab - 1 is even and TMA-eligible)."""
    ld = kl + ku + 2 * EBV_BAND_PAD + 1
    return ld if ld % 2 == 1 else ld + 1


def band_pack(A: torch.Tensor, kl: int, ku: int, ldab: int | None = None) -> torch.Tensor:
    """Compact band storage of a dense (n, n) A (layout of include/ebv.h:
    a_ij at AB[PAD + ku + i - j, j]); returns AB as a (n, ldab) tensor whose
    row j is column j of the (ldab x n) column-major storage.  Layout only."""
    n = A.shape[0]
    ldab = ldab or band_ld(kl, ku)
    AB = torch.zeros(n, ldab, dtype=A.dtype, device=A.device)
    j = torch.arange(n, device=A.device)
    for d in range(-ku, kl + 1):   # diagonal d = i - j
        jj = j[(j + d >= 0) & (j + d < n)]
        AB[jj, EBV_BAND_PAD + ku + d] = A[jj + d, jj]
    return AB


def band_unpack(AB: torch.Tensor, n: int, kl: int, ku: int) -> torch.Tensor:
    """Dense (n, n) matrix holding the band of AB (zeros elsewhere).  Layout only."""
    A = torch.zeros(n, n, dtype=AB.dtype, device=AB.device)
    j = torch.arange(n, device=AB.device)
    for d in range(-ku, kl + 1):
        jj = j[(j + d >= 0) & (j + d < n)]
        A[jj + d, jj] = AB[jj, EBV_BAND_PAD + ku + d]
    return A


def lu_factor_band(AB: torch.Tensor, n: int, kl: int, ku: int, tau: float = 0.0, ctx: Context | None = None):
    """In-place LU of a band-stored matrix (AB from band_pack: (n, ldab),
    contiguous); returns (AB, info)."""
    _require(AB, "AB")
    if not AB.is_contiguous() or AB.shape[0] != n:
        raise EbvError("AB must be a contiguous (n, ldab) tensor (band_pack layout)")
    ctx = ctx or default_context(AB.device.index or 0)
    info = torch.zeros((), dtype=torch.int64, device=AB.device)
    _check(ebv_lu_factor_band(ctx.handle, n, kl, ku, AB.data_ptr(), AB.shape[1], float(tau), info.data_ptr(),
                              _stream_handle(AB.device)), "ebv_lu_factor_band")
    return AB, info


def lu_solve_band(AB: torch.Tensor, B: torch.Tensor, kl: int, ku: int, ctx: Context | None = None):
    """X from band-stored factors (AB as returned by lu_factor_band); B (n,) or (n, nrhs)."""
    _require(AB, "AB")
    n = AB.shape[0]
    ctx = ctx or default_context(AB.device.index or 0)
    vec = B.dim() == 1
    X = B.reshape(n, -1).mT.contiguous().mT.clone()
    _check(ebv_lu_solve_band(ctx.handle, n, kl, ku, AB.data_ptr(), AB.shape[1], X.data_ptr(), max(n, 1),
                             X.shape[1], _stream_handle(AB.device)), "ebv_lu_solve_band")
    return X[:, 0] if vec else X


def ebv_lu_factor_host(ctx, n, hA, ldh, A, lda, tau, d_info, stream):
    return lib().ebv_lu_factor_host(ctx, n, hA, ldh, A, lda, tau, d_info, stream)


def ebv_normalize_unit_diagonal(ctx, n, A, lda, B, ldb, nrhs, d_scales, d_info, stream):
    return lib().ebv_normalize_unit_diagonal(ctx, n, A, lda, B, ldb, nrhs, d_scales, d_info, stream)


def ebv_lu_to_ldu(ctx, n, LU, lda, d_D, stream):
    return lib().ebv_lu_to_ldu(ctx, n, LU, lda, d_D, stream)


def ebv_stats_timeline(ctx, out, max_records):
    return lib().ebv_stats_timeline(ctx, out, max_records)


def ebv_stats_enable(ctx, enable):
    return lib().ebv_stats_enable(ctx, enable)


def ebv_stats_reset(ctx):
    return lib().ebv_stats_reset(ctx)


def ebv_stats_get(ctx, kclass, launches, ms, flops, bytes_):
    return lib().ebv_stats_get(ctx, kclass, launches, ms, flops, bytes_)


def ebv_update(ctx, M, N, K, A, lda, B, ldb, C, ldc, stream):
    return lib().ebv_update(ctx, M, N, K, A, lda, B, ldb, C, ldc, stream)


def update(C: torch.Tensor, A: torch.Tensor, B: torch.Tensor, ctx: Context | None = None):
    """C <- C - A @ B in place (Eq 6-c rank-k update); all column-major CUDA float64."""
    for t, nm in ((C, "C"), (A, "A"), (B, "B")):
        _require(t, nm)
        if _colmajor_ld(t) < 0:
            raise EbvError(f"{nm} must be column-major")
    M, N = C.shape
    K = A.shape[1]
    ctx = ctx or default_context(C.device.index or 0)
    _check(ebv_update(ctx.handle, M, N, K, A.data_ptr(), max(_colmajor_ld(A), 1), B.data_ptr(),
                      max(_colmajor_ld(B), 1), C.data_ptr(), max(_colmajor_ld(C), 1), _stream_handle(C.device)),
           "ebv_update")
    return C


def ebv_plan_owner_map(n: int, workers: int):
    out = (ctypes.c_int32 * max(n, 1))()
    _check(lib().ebv_plan_owner_map(n, workers, out), "ebv_plan_owner_map")
    return list(out)[:n]


def ebv_plan_units(n: int, workers: int):
    m = max(n - 1, 1)
    arrs = [(ctypes.c_int32 * m)() for _ in range(5)]
    _check(lib().ebv_plan_units(n, workers, *arrs), "ebv_plan_units")
    t0, k0, t1, k1, own = (list(a)[: n - 1] for a in arrs)
    tri = "LU"
    units = [((tri[a], b), (tri[c], d)) for a, b, c, d in zip(t0, k0, t1, k1)]
    return units, own


def ebv_block_owner(J, N, nranks, layout=EBV_LAYOUT_CYCLIC) -> int:
    return lib().ebv_block_owner(J, N, nranks, layout)


def ebv_launch_count(ctx) -> int:
    return lib().ebv_launch_count(ctx)


def ebv_set_debug(device: int, flags: int, spin_timeout_s: float = 60.0):
    return lib().ebv_set_debug(device, flags, spin_timeout_s)


def set_debug(flags: int = 0, spin_timeout_s: float = 60.0, device: int = 0):
    """Debug knobs of include/ebv.h (EBV_DEBUG_FORCE_EXACT: every verified
    quotient takes its true-division redo branch; EBV_DEBUG_JITTER: random
    sleeps before cross-CTA flag releases; a bound on flag waits)."""
    _check(ebv_set_debug(device, flags, spin_timeout_s), "ebv_set_debug")


def load_nccl():
    """Make the NCCL that torch ships visible to libebv's dlopen (global)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for d in (spec.submodule_search_locations if spec else []) or []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ.setdefault("EBV_NCCL_LIB", p)
            ctypes.CDLL(p, mode=ctypes.RTLD_GLOBAL)
            return p
    return None


def ebv_get_unique_id() -> bytes:
    load_nccl()
    buf = ctypes.create_string_buffer(128)
    _check(lib().ebv_get_unique_id(buf), "ebv_get_unique_id")
    return buf.raw


def ebv_create_dist(device: int, uid: bytes, rank: int, nranks: int, nb: int = 256,
                    layout: int = EBV_LAYOUT_CYCLIC) -> int:
    load_nccl()
    h = _vp()
    _check(lib().ebv_create_dist(ctypes.byref(h), device, ctypes.create_string_buffer(uid, 128), rank, nranks,
                                 nb, layout), "ebv_create_dist")
    return h.value


def ebv_dist_nranks(ctx) -> int:
    return lib().ebv_dist_nranks(ctx)


def ebv_dist_local_blocks(n: int, nb: int, rank: int, nranks: int, layout: int = EBV_LAYOUT_CYCLIC):
    """(blocks owned by `rank` in ascending order, local slab width)."""
    nbk, cols = _i64(), _i64()
    _check(lib().ebv_dist_local_blocks(n, nb, rank, nranks, layout, None, 0, ctypes.byref(nbk),
                                       ctypes.byref(cols)), "ebv_dist_local_blocks")
    arr = (ctypes.c_int64 * max(nbk.value, 1))()
    _check(lib().ebv_dist_local_blocks(n, nb, rank, nranks, layout, arr, nbk.value, ctypes.byref(nbk),
                                       ctypes.byref(cols)), "ebv_dist_local_blocks")
    return list(arr)[: nbk.value], cols.value


def dist_local_columns(n: int, nb: int, rank: int, nranks: int, layout: int = EBV_LAYOUT_CYCLIC):
    """Global column indices of rank's slab, in slab order."""
    blocks, _ = ebv_dist_local_blocks(n, nb, rank, nranks, layout)
    cols = []
    for J in blocks:
        cols.extend(range(J * nb, min(n, (J + 1) * nb)))
    return cols


def ebv_lu_factor_dist(ctx, n, A_local, lda, tau, d_info, stream):
    return lib().ebv_lu_factor_dist(ctx, n, A_local, lda, tau, d_info, stream)


def ebv_lu_solve_dist(ctx, n, LU_local, lda, B, ldb, nrhs, stream):
    return lib().ebv_lu_solve_dist(ctx, n, LU_local, lda, B, ldb, nrhs, stream)


def ebv_lu_factor_dist_emulated(ctx, n, nranks, nb, layout, slab_ptrs, lda, tau, d_info, stream):
    arr = (ctypes.c_void_p * nranks)(*slab_ptrs)
    return lib().ebv_lu_factor_dist_emulated(ctx, n, nranks, nb, layout, arr, lda, tau, d_info, stream)


def ebv_lu_solve_dist_emulated(ctx, n, nranks, nb, layout, slab_ptrs, lda, B, ldb, nrhs, stream):
    arr = (ctypes.c_void_p * nranks)(*slab_ptrs)
    return lib().ebv_lu_solve_dist_emulated(ctx, n, nranks, nb, layout, arr, lda, B, ldb, nrhs, stream)


# ------------------------------------------------------------------ tensor helpers
def _stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Context:
    """Owns an ebv_context_t on one CUDA device."""

    def __init__(self, device: int | torch.device = 0, path: int = EBV_PATH_AUTO, leaf: int = 0):
        if isinstance(device, torch.device):
            device = device.index or 0
        if not torch.cuda.is_available():
            raise EbvError("paper_1907_05767_b200 needs a CUDA device (no CPU fallback)")
        self.device = int(device)
        self.handle = ebv_create(self.device)
        _check(ebv_set_path(self.handle, path), "ebv_set_path")
        _check(ebv_set_leaf(self.handle, leaf), "ebv_set_leaf")

    def set_path(self, path: int):
        _check(ebv_set_path(self.handle, path), "ebv_set_path")

    def set_leaf(self, leaf: int):
        _check(ebv_set_leaf(self.handle, leaf), "ebv_set_leaf")

    def set_block(self, nb: int):
        _check(ebv_set_block(self.handle, nb), "ebv_set_block")

    def block_width(self, n: int) -> int:
        """Column block width the blocked schedule uses at order n (-1: recursive)."""
        return int(ebv_block_width(self.handle, n))

    def set_lookahead(self, on: bool):
        _check(ebv_set_lookahead(self.handle, on), "ebv_set_lookahead")

    def set_graphs(self, on: bool):
        _check(ebv_set_graphs(self.handle, on), "ebv_set_graphs")

    def set_vector_ctas(self, ctas: int):
        _check(ebv_set_vector_ctas(self.handle, ctas), "ebv_set_vector_ctas")

    def stats_enable(self, on: bool = True):
        _check(lib().ebv_stats_enable(self.handle, 1 if on else 0), "ebv_stats_enable")

    def stats_reset(self):
        _check(lib().ebv_stats_reset(self.handle), "ebv_stats_reset")

    def stats(self) -> dict:
        out = {}
        for c, name in enumerate(KCLASSES):
            n, ms, fl, by = _i64(), _d(), _d(), _d()
            _check(lib().ebv_stats_get(self.handle, c, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl),
                                       ctypes.byref(by)), "ebv_stats_get")
            out[name] = {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
        return out

    def timeline(self) -> list:
        """Recorded launches since the last stats reset:
        [(class name, start ms, end ms, on the lookahead side stream)]."""
        L = lib()
        n = L.ebv_stats_timeline(self.handle, None, 0)
        if n < 0:
            raise EbvError("ebv_stats_timeline failed")
        buf = (ctypes.c_double * (3 * max(n, 1)))()
        n = L.ebv_stats_timeline(self.handle, buf, n)
        return [(KCLASSES[int(buf[3 * i]) & 0xFF], buf[3 * i + 1], buf[3 * i + 2], bool(int(buf[3 * i]) >> 8))
                for i in range(n)]

    def launch_count(self) -> int:
        return ebv_launch_count(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            ebv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _colmajor_ld(t: torch.Tensor) -> int:
    """Leading dimension if t (logical [rows, cols]) is column-major-strided
    with ld >= rows, else -1."""
    if t.dim() != 2:
        return -1
    rows, cols = t.shape
    if cols <= 1:
        return max(rows, 1) if (t.stride(0) == 1 or rows <= 1) else -1
    if t.stride(0) != 1 and rows > 1:
        return -1
    return t.stride(1) if t.stride(1) >= max(rows, 1) else -1


def colmajor_copy(t: torch.Tensor) -> torch.Tensor:
    """A fresh column-major (Fortran-ordered) copy of a 2-D tensor."""
    return t.mT.clone(memory_format=torch.contiguous_format).mT


def _require(t: torch.Tensor, what: str):
    if not t.is_cuda or t.dtype != torch.float64:
        raise EbvError(f"{what} must be a CUDA float64 tensor")


def lu_factor(A: torch.Tensor, tau: float = 0.0, ctx: Context | None = None, inplace: bool = False):
    """A = LU without pivoting (Eq 6).  A: (n, n) CUDA float64, logical
    indexing.  Returns (LU, info): LU is the column-major packed L\\U (A
    itself when inplace=True, which needs column-major A), info a 0-dim int64
    CUDA tensor (0 or the first failing 1-based step)."""
    _require(A, "A")
    n = A.shape[0]
    if A.dim() != 2 or A.shape[1] != n:
        raise EbvError("A must be square")
    ctx = ctx or default_context(A.device.index or 0)
    if inplace:
        if _colmajor_ld(A) < 0:
            raise EbvError("inplace lu_factor needs a column-major A (A.mT contiguous)")
        LU = A
    else:
        LU = colmajor_copy(A)
    info = torch.zeros((), dtype=torch.int64, device=A.device)
    _check(ebv_lu_factor(ctx.handle, n, LU.data_ptr(), max(_colmajor_ld(LU), 1), float(tau), info.data_ptr(),
                         _stream_handle(A.device)), "ebv_lu_factor")
    return LU, info


def lu_solve(LU: torch.Tensor, B: torch.Tensor, ctx: Context | None = None, inplace: bool = False):
    """X from LY = B then UX = Y (Eq 1).  B: (n,) or (n, nrhs) CUDA float64.
    Returns X (B itself when inplace=True and B is column-major)."""
    _require(LU, "LU")
    _require(B, "B")
    n = LU.shape[0]
    ctx = ctx or default_context(LU.device.index or 0)
    vec = B.dim() == 1
    B2 = B.reshape(n, 1) if vec else B
    if inplace and _colmajor_ld(B2) > 0:
        X = B2
    else:
        X = colmajor_copy(B2)
    LUc = LU if _colmajor_ld(LU) > 0 else colmajor_copy(LU)
    _check(ebv_lu_solve(ctx.handle, n, LUc.data_ptr(), max(_colmajor_ld(LUc), 1), X.data_ptr(),
                        max(_colmajor_ld(X), 1), X.shape[1], _stream_handle(LU.device)), "ebv_lu_solve")
    if vec:
        return X.reshape(n)
    return X


def lu_factor_batched(At: torch.Tensor, Bt: torch.Tensor | None = None, tau: float = 0.0,
                      ctx: Context | None = None):
    """In place on per-system column-major storage: At (batch, n, n) with
    At[s, j, i] = a^(s)_ij (contiguous), Bt (batch, nrhs, n) with Bt[s, r, i]
    = b^(s)_i,r (contiguous) or None.  Returns the int32 info tensor."""
    _require(At, "At")
    if not At.is_contiguous():
        raise EbvError("At must be contiguous (batch, n, n) column-major storage")
    batch, n, _ = At.shape
    ctx = ctx or default_context(At.device.index or 0)
    info = torch.zeros(batch, dtype=torch.int32, device=At.device)
    if Bt is not None:
        _require(Bt, "Bt")
        if not Bt.is_contiguous():
            raise EbvError("Bt must be contiguous (batch, nrhs, n)")
        nrhs = Bt.shape[1]
        bptr, ldb, sb = Bt.data_ptr(), max(n, 1), n * nrhs
    else:
        nrhs, bptr, ldb, sb = 0, None, max(n, 1), 0
    _check(ebv_lu_factor_batched(ctx.handle, n, At.data_ptr(), max(n, 1), n * n, batch, bptr, ldb, sb, nrhs,
                                 float(tau), info.data_ptr(), _stream_handle(At.device)), "ebv_lu_factor_batched")
    return info


def lu_factor_host(hA: torch.Tensor, tau: float = 0.0, ctx: Context | None = None, device: int = 0,
                   out: torch.Tensor | None = None):
    """A = LU of a host-resident matrix (ebv_lu_factor_host): hA (n, n) CPU
    float64 in logical indexing, column-major storage (hA.mT contiguous;
    pinned memory lets the block copies overlap the factorization).  Returns
    (LU, info) on cuda:device (LU column-major; `out` may supply it)."""
    if hA.device.type != "cpu" or hA.dtype != torch.float64 or hA.dim() != 2:
        raise EbvError("hA must be a 2-D float64 CPU tensor")
    n = hA.shape[0]
    ldh = _colmajor_ld(hA)
    if ldh < 0:
        raise EbvError("hA must be column-major (hA.mT contiguous)")
    ctx = ctx or default_context(device)
    dev = torch.device("cuda", ctx.device)
    LU = out if out is not None else torch.empty(n, n, dtype=torch.float64, device=dev).mT
    info = torch.zeros((), dtype=torch.int64, device=dev)
    _check(ebv_lu_factor_host(ctx.handle, n, hA.data_ptr(), max(ldh, 1), LU.data_ptr(), max(_colmajor_ld(LU), 1),
                              float(tau), info.data_ptr(), _stream_handle(dev)), "ebv_lu_factor_host")
    return LU, info


def normalize_unit_diagonal(A: torch.Tensor, B: torch.Tensor | None = None, ctx: Context | None = None):
    """Row i of A (and of B) divided by a_ii (Eq 2).  A: (n, n)
    CUDA float64, logical indexing; B: (n,) or (n, nrhs) or None.  Returns
    (A', B' or None, scales, info) with new column-major A' / B'."""
    _require(A, "A")
    n = A.shape[0]
    ctx = ctx or default_context(A.device.index or 0)
    Ac = A.mT.contiguous().mT.clone() if _colmajor_ld(A) < 0 else A.clone()
    Bc, nrhs = None, 0
    if B is not None:
        _require(B, "B")
        B2 = B.reshape(n, -1)
        Bc = B2.mT.contiguous().mT.clone()
        nrhs = Bc.shape[1]
    scales = torch.empty(n, dtype=torch.float64, device=A.device)
    info = torch.zeros((), dtype=torch.int64, device=A.device)
    _check(lib().ebv_normalize_unit_diagonal(ctx.handle, n, Ac.data_ptr(), max(_colmajor_ld(Ac), 1),
                                             Bc.data_ptr() if Bc is not None else None, max(n, 1), nrhs,
                                             scales.data_ptr(), info.data_ptr(), _stream_handle(A.device)),
           "ebv_normalize_unit_diagonal")
    if Bc is not None and B.dim() == 1:
        Bc = Bc[:, 0]
    return Ac, Bc, scales, info


def lu_to_ldu(LU: torch.Tensor, ctx: Context | None = None):
    """LDU form of a packed LU (Eq 3): returns (LDU, D) — a column-major copy
    with U' = D^-1 U in its strict upper triangle, and D = diag(U)."""
    _require(LU, "LU")
    n = LU.shape[0]
    ctx = ctx or default_context(LU.device.index or 0)
    Lc = LU.mT.contiguous().mT.clone() if _colmajor_ld(LU) < 0 else LU.clone()
    D = torch.empty(n, dtype=torch.float64, device=LU.device)
    _check(lib().ebv_lu_to_ldu(ctx.handle, n, Lc.data_ptr(), max(_colmajor_ld(Lc), 1), D.data_ptr(),
                               _stream_handle(LU.device)), "ebv_lu_to_ldu")
    return Lc, D


def lu_solve_batched(LUt: torch.Tensor, Bt: torch.Tensor, ctx: Context | None = None) -> torch.Tensor:
    """Solve-only for systems factored by lu_factor_batched: LUt (batch, n, n)
    packed per-system column-major storage (read only), Bt (batch, nrhs, n)
    overwritten with X.  Returns Bt."""
    _require(LUt, "LUt")
    _require(Bt, "Bt")
    if not LUt.is_contiguous() or not Bt.is_contiguous():
        raise EbvError("LUt (batch, n, n) and Bt (batch, nrhs, n) must be contiguous")
    batch, n, _ = LUt.shape
    nrhs = Bt.shape[1]
    ctx = ctx or default_context(LUt.device.index or 0)
    _check(ebv_lu_solve_batched(ctx.handle, n, LUt.data_ptr(), max(n, 1), n * n, batch, Bt.data_ptr(), max(n, 1),
                                n * nrhs, nrhs, _stream_handle(LUt.device)), "ebv_lu_solve_batched")
    return Bt
