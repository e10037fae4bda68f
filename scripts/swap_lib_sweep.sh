# run the RHS sweep with the in-tree library, then with an alternative build
python scripts/solve_rhs_sweep.py 8192,32768 2>&1 | grep -E '"nrhs": (1|16|64),' | cut -c1-70
cp paper_1907_05767_b200/libebv.so /tmp/libebv_orig.so
cp "$1" paper_1907_05767_b200/libebv.so
echo alt
python scripts/solve_rhs_sweep.py 8192,32768 2>&1 | grep -E '"nrhs": (1|16|64),' | cut -c1-70
cp /tmp/libebv_orig.so paper_1907_05767_b200/libebv.so
