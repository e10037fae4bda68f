"""Per-launch timeline of one blocked factorization (stats mode) and where
the time goes: per column step, the main-stream span vs the GEMM work."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import json
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--nb", type=int, default=0)
ap.add_argument("--out", default="")
ap.add_argument("--no-lookahead", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda:0")
d = ebv_inputs.generate(a.n, seed=1, device=dev)
A0 = d["At"]
ctx = ebv.Context(0)
ctx.set_block(a.nb)
if a.no_lookahead:
    ctx.set_lookahead(False)
s = torch.cuda.Stream(dev)
info = torch.zeros((), dtype=torch.int64, device=dev)
with torch.cuda.stream(s):
    for rep in range(3):
        A = A0.clone()
        torch.cuda.synchronize()
        if rep == 2:
            ctx.stats_reset()
            ctx.stats_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ebv.ebv_lu_factor(ctx.handle, a.n, A.data_ptr(), a.n, 0.0, info.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        print("rep", rep, "ms", e0.elapsed_time(e1), "stats" if rep == 2 else "")
tl = ctx.timeline()
ctx.stats_enable(False)
tot = {}
for cls, t0, t1, side in tl:
    k = (cls, side)
    tot.setdefault(k, [0, 0.0])
    tot[k][0] += 1
    tot[k][1] += t1 - t0
end = max(t1 for _, _, t1, _ in tl)
print("span ms", end, "launches", len(tl))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print("  %-10s side=%d launches=%5d busy_ms=%.3f avg_us=%.1f" % (k[0], k[1], v[0], v[1], 1e3 * v[1] / v[0]))
# per-launch durations of the small kernels in the last steps (standalone when no lookahead)
last = [(c, round(1e3 * (t1 - t0), 1)) for c, t0, t1, sd in tl[-24:]]
print("last launches (class, us):", last)
# main-stream idle gaps (between consecutive main-stream launches)
main = sorted([(t0, t1, c) for c, t0, t1, sd in tl if not sd])
gap = 0.0
big = []
for (a0, a1, c0), (b0, b1, c1) in zip(main, main[1:]):
    g = b0 - a1
    if g > 0:
        gap += g
        big.append((g, a1, c0, c1))
print("main-stream idle ms", gap)
for g, t, c0, c1 in sorted(big, reverse=True)[:15]:
    print("   gap %.3f ms at %.3f after %s before %s" % (g, t, c0, c1))
if a.out:
    json.dump(tl, open(a.out, "w"))
