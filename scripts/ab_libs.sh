# A/B: run a command with the in-tree library and with each alternative build
# given as arguments (paths to libebv.so); restores the in-tree one after.
CMD="$1"; shift
cp paper_1907_05767_b200/libebv.so /tmp/libebv_orig.so
echo "== in-tree"; eval "$CMD"
for L in "$@"; do
  cp "$L" paper_1907_05767_b200/libebv.so
  echo "== $L"; eval "$CMD"
done
cp /tmp/libebv_orig.so paper_1907_05767_b200/libebv.so
