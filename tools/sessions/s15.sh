# 4-blocks/SM geometries: u32+u8 (256x32), u64 keys-only (256x24), u32+u64 (256x16)
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in v1 v2 v3; do
  echo "== $v parity: $(ONESWEEP_B200_LIB=$V/$v.so timeout 900 python -m pytest tests/test_gpu_value_widths.py -x -q -k 2e26 2>&1 | tail -1)"
done
for v in base v1 v2 v3; do echo "== $v"; ONESWEEP_B200_LIB=$V/$v.so timeout 600 python tools/value_widths.py; done
