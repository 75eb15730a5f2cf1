# time alternative builds of librfxc.so kept in variants/ (scratch)
cd "${GRAFT_REPO_ROOT:-.}"
cp paper_2511_19493_b200/_build/librfxc.so /tmp/librfxc_orig.so
for f in variants/*.so; do
  cp $f paper_2511_19493_b200/_build/librfxc.so
  echo "== $f"; eval "${CMD:-RFXC_SKETCH_TIMING=1 python scripts/path_probe.py 64 2>&1 | grep 'sketch. pass' | tail -1}"
done
cp /tmp/librfxc_orig.so paper_2511_19493_b200/_build/librfxc.so
