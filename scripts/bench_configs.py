"""Per-config measurements for BASELINE.json configs C1, C2, C3, C5 (C4 is
bench.py's headline).  CUDA-event timing on the launching stream, warm-up 3,
median of 5, inputs restored from pristine device copies outside the events,
all on one non-default stream (so repeated factorizations replay a graph).
One JSON line per measurement."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import statistics

import torch

import ebv_inputs
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
# a non-default stream for everything (torch copies included): the library
# captures the blocked factor schedule into a CUDA graph on the second call
# with identical arguments there and replays it afterwards
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
sh = stream.cuda_stream
PEAK_TF = 37.116
HBM = 6538.6


def timeit(prep, fn, reps=5, warm=3):
    ts = []
    for r in range(warm + reps):
        prep()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts), max(ts)


def emit(**kw):
    print(json.dumps(kw), flush=True)


ctx = ebv.Context(0)
info = torch.zeros((), dtype=torch.int64, device=dev)

# ---------------- C1 / C2 / C3 dense factor (+ solve)
for cfg, n, nrhs in (("C1", 64, 1), ("C2", 1024, 1), ("C3", 8192, 16)):
    d = ebv_inputs.generate(n, seed=1, nrhs=nrhs, device=dev)
    A0, B0 = d["At"], d["B"].T.clone(memory_format=torch.contiguous_format)
    Aw, Bw = torch.empty_like(A0), torch.empty_like(B0)
    fl = 2.0 / 3.0 * n ** 3
    paths = [("blocked", ebv.EBV_PATH_BLOCKED)]
    if n <= 1536:
        paths += [("vector_ebvpair", ebv.EBV_PATH_VECTOR), ("vector_cyclic", -1)]
    for name, path in paths:
        if path == -1:
            ctx.set_path(ebv.EBV_PATH_VECTOR)
            C = min(148, n // 2) if n >= 2 else 1
            ctx.set_vector_ctas(-C)
        else:
            ctx.set_path(path)
            ctx.set_vector_ctas(0)
        med, lo, hi = timeit(lambda: Aw.copy_(A0),
                             lambda: ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), sh))
        ok = int(info) == 0
        rec = {"config": cfg, "n": n, "what": "factor", "path": name, "ms": med, "ms_min": lo, "ms_max": hi,
               "gflops": fl / med / 1e6, "frac_fp64_peak": fl / med / 1e9 / PEAK_TF, "info_ok": ok}
        if name.startswith("vector"):
            rec["us_per_step"] = 1e3 * med / max(n - 1, 1)
        emit(**rec)
    ctx.set_path(ebv.EBV_PATH_AUTO)
    ctx.set_vector_ctas(0)
    Aw.copy_(A0)
    ebv.ebv_lu_factor(ctx.handle, n, Aw.data_ptr(), n, 0.0, info.data_ptr(), sh)
    med, lo, hi = timeit(lambda: Bw.copy_(B0),
                         lambda: ebv.ebv_lu_solve(ctx.handle, n, Aw.data_ptr(), n, Bw.data_ptr(), n, nrhs, sh))
    err = (Bw.T - d["X"]).abs().max().item()
    emit(config=cfg, n=n, nrhs=nrhs, what="solve", ms=med, ms_min=lo, ms_max=hi,
         gbs=8.0 * n * n / med / 1e6, frac_hbm=8.0 * n * n / med / 1e6 / HBM, max_err=err)
    # context: cuSOLVER no-pivot getrf (library comparator, never on the product path)
    if n >= 1024:
        A = A0.T.contiguous()
        med, lo, hi = timeit(lambda: None, lambda: torch.linalg.lu_factor(A, pivot=False))
        emit(config=cfg, n=n, what="factor", path="cusolver_getrf_nopivot(context)", ms=med,
             gflops=fl / med / 1e6)
    del d, A0, B0, Aw, Bw

# ---------------- C5 batched
batch = 100_000
db = ebv_inputs.generate_batched(batch, 32, seed=1, nrhs=1, device=dev)
A0 = db["At"]
B0 = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
Aw, Bw = torch.empty_like(A0), torch.empty_like(B0)
binfo = torch.zeros(batch, dtype=torch.int32, device=dev)


def prep():
    Aw.copy_(A0)
    Bw.copy_(B0)


med, lo, hi = timeit(prep, lambda: ebv.ebv_lu_factor_batched(ctx.handle, 32, Aw.data_ptr(), 32, 1024, batch,
                                                             Bw.data_ptr(), 32, 32, 1, 0.0, binfo.data_ptr(), sh))
by = batch * (2 * 32 * 32 * 8 + 2 * 32 * 8 + 4)
emit(config="C5", batch=batch, n=32, what="batched factor+solve", ms=med, ms_min=lo, ms_max=hi,
     gbs=by / med / 1e6, frac_hbm=by / med / 1e6 / HBM, systems_per_s=batch / med * 1e3,
     max_err=(Bw.transpose(1, 2) - db["X"]).abs().max().item(), bytes=by)

# ---------------- f1: factor once, solve many (batched solve-only on the factors above)
for nr in (1, 16):
    Bn = torch.randn(batch, nr, 32, dtype=torch.float64, device=dev)
    Bw2 = torch.empty_like(Bn)
    med, lo, hi = timeit(lambda: Bw2.copy_(Bn),
                         lambda: ebv.ebv_lu_solve_batched(ctx.handle, 32, Aw.data_ptr(), 32, 1024, batch,
                                                          Bw2.data_ptr(), 32, 32 * nr, nr, sh))
    by = batch * (32 * 32 * 8 + 2 * 32 * nr * 8)
    emit(config="C5-solve-only", batch=batch, n=32, nrhs=nr, what="batched solve (pre-factored)", ms=med,
         ms_min=lo, ms_max=hi, gbs=by / med / 1e6, frac_hbm=by / med / 1e6 / HBM,
         systems_per_s=batch / med * 1e3, bytes=by)

# ---------------- f2: batched medium systems (n = 64, CTA per system)
db = ebv_inputs.generate_batched(batch, 64, seed=1, nrhs=1, device=dev)
A64 = db["At"]
B64 = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
Aw64, Bw64 = torch.empty_like(A64), torch.empty_like(B64)


def prep64():
    Aw64.copy_(A64)
    Bw64.copy_(B64)


med, lo, hi = timeit(prep64, lambda: ebv.ebv_lu_factor_batched(ctx.handle, 64, Aw64.data_ptr(), 64, 64 * 64, batch,
                                                                Bw64.data_ptr(), 64, 64, 1, 0.0, binfo.data_ptr(), sh))
by = batch * (2 * 64 * 64 * 8 + 2 * 64 * 8 + 4)
emit(config="f2-batched64", batch=batch, n=64, what="batched factor+solve", ms=med, ms_min=lo, ms_max=hi,
     gbs=by / med / 1e6, frac_hbm=by / med / 1e6 / HBM, systems_per_s=batch / med * 1e3,
     max_err=(Bw64.transpose(1, 2) - db["X"]).abs().max().item(), bytes=by)
del db, A64, B64, Aw64, Bw64

# ---------------- f3: unit-diagonal normalization and LDU form at n = 32768 (HBM-bound)
del A0, B0, Aw, Bw
n = 32768
d = ebv_inputs.generate(n, seed=1, nrhs=1, device=dev)
A0 = d["At"]
Aw = torch.empty_like(A0)
Bw = d["B"].T.clone(memory_format=torch.contiguous_format)
scales = torch.empty(n, dtype=torch.float64, device=dev)
info1 = torch.zeros((), dtype=torch.int64, device=dev)
med, lo, hi = timeit(lambda: Aw.copy_(A0),
                     lambda: ebv.ebv_normalize_unit_diagonal(ctx.handle, n, Aw.data_ptr(), n, Bw.data_ptr(), n, 1,
                                                             scales.data_ptr(), info1.data_ptr(), sh))
by = 16.0 * n * n + 16.0 * n
emit(config="f3-normalize", n=n, what="unit-diagonal normalization (A and b)", ms=med, ms_min=lo, ms_max=hi,
     gbs=by / med / 1e6, frac_hbm=by / med / 1e6 / HBM)
D = torch.empty(n, dtype=torch.float64, device=dev)
med, lo, hi = timeit(lambda: Aw.copy_(A0),
                     lambda: ebv.ebv_lu_to_ldu(ctx.handle, n, Aw.data_ptr(), n, D.data_ptr(), sh))
by = 16.0 * n * (n - 1) / 2
emit(config="f3-ldu", n=n, what="LDU form (strict upper / pivot)", ms=med, ms_min=lo, ms_max=hi,
     gbs=by / med / 1e6, frac_hbm=by / med / 1e6 / HBM)

# ---------------- f2: batched medium orders (64 < n <= 512: batched blocked schedule)
for nm, bm in ((128, 20000), (256, 4000), (512, 800)):
    dbm = ebv_inputs.generate_batched(bm, nm, seed=2, nrhs=1, device=dev)
    Am = dbm["At"]
    Bm = dbm["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format)
    Xm = dbm["X"]
    Awm, Bwm = torch.empty_like(Am), torch.empty_like(Bm)
    infom = torch.zeros(bm, dtype=torch.int32, device=dev)
    del dbm

    def prepm():
        Awm.copy_(Am)
        Bwm.copy_(Bm)

    med, lo, hi = timeit(prepm, lambda: ebv.ebv_lu_factor_batched(ctx.handle, nm, Awm.data_ptr(), nm, nm * nm, bm,
                                                                  Bwm.data_ptr(), nm, nm, 1, 0.0, infom.data_ptr(), sh))
    fl = bm * (2.0 / 3.0 * nm ** 3 + 2.0 * nm * nm)
    emit(config="f2-batched-medium", batch=bm, n=nm, what="batched factor+solve (blocked, all systems per launch)",
         ms=med, ms_min=lo, ms_max=hi, tflops=fl / med / 1e9, frac_fp64_peak=fl / med / 1e9 / PEAK_TF,
         systems_per_s=bm / med * 1e3, info_ok=not infom.any().item(),
         max_err=(Bwm.transpose(1, 2) - Xm).abs().max().item())
    del Am, Bm, Awm, Bwm, Xm

# ---------------- f4: banded / 2D five-point stencil (zero-skip), dense storage
for m in (128, 256):
    n = m * m
    d = ebv_inputs.generate(n, seed=1, nrhs=1, device=dev, stencil_m=m)
    A0 = d["At"]
    Aw = torch.empty_like(A0)
    Bs = d["B"].T.clone(memory_format=torch.contiguous_format)
    Bw = torch.empty_like(Bs)
    X = d["X"]
    del d
    med, lo, hi = timeit(lambda: Aw.copy_(A0),
                         lambda: ebv.ebv_lu_factor_banded(ctx.handle, n, m, m, Aw.data_ptr(), n, 0.0, info.data_ptr(),
                                                          sh))
    fl = 2.0 * n * m * m        # band LU flops ~ 2 n kl ku
    emit(config="f4-stencil", n=n, m=m, kl=m, ku=m, what="banded factor (zero-skip)", ms=med, ms_min=lo, ms_max=hi,
         gflops_band=fl / med / 1e6, info_ok=int(info) == 0)
    med2, lo2, hi2 = timeit(lambda: Bw.copy_(Bs),
                            lambda: ebv.ebv_lu_solve_banded(ctx.handle, n, m, m, Aw.data_ptr(), n, Bw.data_ptr(), n, 1,
                                                            sh))
    emit(config="f4-stencil", n=n, m=m, what="banded solve (zero-skip)", ms=med2, ms_min=lo2, ms_max=hi2,
         max_err=(Bw.T - X).abs().max().item())
    del A0, Aw, Bs, Bw, X

# ---------------- f4: compact band storage (ebv_lu_factor_band): memory ~ n (kl + ku)
for n, kl, ku in ((65536, 256, 256), (262144, 128, 128), (1048576, 64, 64)):
    ld = ebv.band_ld(kl, ku)
    g = ebv_inputs.generate_band(n, kl, ku, ebv.EBV_BAND_PAD, ld, seed=1, device=dev)
    AB0 = g["AB"]
    ABw = torch.empty_like(AB0)
    Bs = g["B"].T.contiguous()
    Bw = torch.empty_like(Bs)
    X = g["X"]
    del g
    med, lo, hi = timeit(lambda: ABw.copy_(AB0),
                         lambda: ebv.ebv_lu_factor_band(ctx.handle, n, kl, ku, ABw.data_ptr(), ld, 0.0,
                                                        info.data_ptr(), sh))
    emit(config="f4-band-storage", n=n, kl=kl, ku=ku, ldab=ld, storage_gb=8.0 * n * ld / 1e9,
         dense_storage_gb=8.0 * n * n / 1e9, what="band factor (compact storage)", ms=med, ms_min=lo, ms_max=hi,
         gflops_band=2.0 * n * kl * ku / med / 1e6, info_ok=int(info) == 0)
    med2, lo2, hi2 = timeit(lambda: Bw.copy_(Bs),
                            lambda: ebv.ebv_lu_solve_band(ctx.handle, n, kl, ku, ABw.data_ptr(), ld, Bw.data_ptr(),
                                                          n, 1, sh))
    emit(config="f4-band-storage", n=n, kl=kl, ku=ku, what="band solve (compact storage)", ms=med2, ms_min=lo2,
         ms_max=hi2, max_err=(Bw.T - X).abs().max().item())
    del AB0, ABw, Bs, Bw, X
