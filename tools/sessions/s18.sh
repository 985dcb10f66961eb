# instruction / wavefront counts of the C2 binning pass with and without pass routing
cd $GRAFT_REPO_ROOT
V=$PWD/paper_2206_01784_b200/_lib/variants
for v in head route; do
  echo "== $v"
  ONESWEEP_B200_LIB=$V/$v.so ncu --metrics smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,gpu__time_duration.sum,launch__registers_per_thread -k regex:binning -s 4 -c 2 \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | grep -E "inst_executed|wavefronts|duration|registers"
done
