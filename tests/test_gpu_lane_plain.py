"""The plain lane map kept for the lane-level EbV comparison (SURVEY §8(a'),
DESIGN §7): `EBV_BATCHED_PLAIN=1` selects one system per warp (lane = row);
its results must be bitwise the oracle's like the paired kernel's.  The
switch is read once per process, so the check runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, ebv_inputs, oracle
import paper_1907_05767_b200 as ebv
dev = torch.device("cuda:0")
ctx = ebv.Context(0)
for n, batch, nrhs in ((32, 300, 1), (20, 41, 1), (32, 65, 0)):
    db = ebv_inputs.generate_batched(batch, n, seed=n + batch, nrhs=1, device=dev)
    At = db["At"].clone()
    Bt = db["B"].transpose(1, 2).clone(memory_format=torch.contiguous_format) if nrhs else None
    info = ebv.lu_factor_batched(At, Bt, ctx=ctx)
    torch.cuda.synchronize()
    a = db["At"].transpose(1, 2).cpu().numpy()
    b = db["B"].cpu().numpy() if nrhs else None
    lu_o, x_o, info_o = oracle.lu_factor_batched(a, b)
    assert np.array_equal(info.cpu().numpy(), info_o)
    assert np.array_equal(At.transpose(1, 2).cpu().numpy().view(np.uint64), lu_o.view(np.uint64))
    if nrhs:
        assert np.array_equal(Bt.transpose(1, 2).cpu().numpy().view(np.uint64), x_o.view(np.uint64))
print("plain lane map bitwise ok")
"""


def test_plain_lane_map_bitwise():
    env = dict(os.environ, EBV_BATCHED_PLAIN="1")
    r = subprocess.run([sys.executable, "-c", SNIPPET, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bitwise ok" in r.stdout
