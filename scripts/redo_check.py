"""Factor time with the verified quotients forced through their true-division
redo (EBV_DEBUG_FORCE_EXACT) vs normal: if they match, the redo path is
being taken anyway.  python scripts/redo_check.py [n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ebv_inputs
import paper_1907_05767_b200 as ebv

dev = torch.device("cuda:0")
for n in [int(x) for x in sys.argv[1:]] or [1024]:
    A0 = ebv_inputs.generate(n, seed=1, device=dev, with_b=False)["At"]
    info = torch.zeros((), dtype=torch.int64, device=dev)
    ctx = ebv.Context(0)
    s = torch.cuda.Stream(dev)
    for force in (0, 1, 0):
        ebv.set_debug(ebv.EBV_DEBUG_FORCE_EXACT if force else 0)
        ts = []
        with torch.cuda.stream(s):
            for r in range(8):
                A = A0.clone()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                ebv.ebv_lu_factor(ctx.handle, n, A.data_ptr(), n, 0.0, info.data_ptr(), s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
        print(n, "force_exact" if force else "normal", sorted(ts)[4])
    ebv.set_debug(0)
