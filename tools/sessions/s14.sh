# TMEM stash for 1/2/8-byte values and wider geometries for the non-benchmark (key, value) widths
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in cur g1 g2; do
  echo "== $v parity: $(ONESWEEP_B200_LIB=$V/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide_values.py -x -q 2>&1 | tail -1)"
done
for v in head cur g1 g2; do
  echo "== $v"; ONESWEEP_B200_LIB=$V/$v.so timeout 600 python tools/value_widths.py
done
