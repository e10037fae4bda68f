"""U12 lookahead schedule (EBV_U12_LA): step K updates block
row K+1 first and the side stream solves U12 of step K+1 while the main
stream updates the rows below.  Per entry the updates are unchanged, so the
factors must stay bitwise the oracle's (Eq 6).  The knob is read
when libebv.so loads, hence the child process; by default it is on only for
n >= 16384, so this forces it on small orders (several panel widths, ragged
tails, banded inputs, CUDA-graph replay)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import ebv_inputs, oracle
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
ctx = ebv.Context(0)
def bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
for n, nb, kl, ku, reps in ((700, 64, None, None, 1), (1537, 128, None, None, 1), (1000, 64, 200, 300, 1),
                            (2048, 256, None, None, 3), (1100, 64, 64, 64, 1)):
    d = ebv_inputs.generate(n, seed=n + nb, device=dev, kl=kl, ku=ku)
    A = d["At"].T
    ctx.set_block(nb)
    for r in range(reps):
        if kl is None:
            LU, info = ebv.lu_factor(A, ctx=ctx)
        else:
            LU, info = ebv.lu_factor_banded(A, kl, ku, ctx=ctx)
        torch.cuda.synchronize()
        lu_o, _ = oracle.lu_factor(A.cpu().numpy())
        assert bits(LU.cpu().numpy(), lu_o), (n, nb, kl, ku, r)
        assert int(info) == 0
print("OK")
"""


@pytest.mark.gpu
def test_u12_lookahead_bitwise():
    env = dict(os.environ, EBV_U12_LA="1")
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]


@pytest.mark.gpu
def test_u12_lookahead_distributed_emulated_bitwise():
    """The distributed schedule's U12 lookahead (ebv_dist.cu), forced on for
    the emulated P-rank tests of tests/test_gpu_dist.py (bitwise against the
    oracle there)."""
    env = dict(os.environ, EBV_U12_LA="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          os.path.join(ROOT, "tests", "test_gpu_dist.py"), "-k", "emulated"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
