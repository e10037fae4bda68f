timeout -s KILL 300 python scripts/check_gemm.py 2>&1 | tail -25
EBV_GEMM_TMA=-1 timeout -s KILL 300 python scripts/check_gemm.py 2>&1 | tail -6
