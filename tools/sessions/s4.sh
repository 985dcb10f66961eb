# PDL between passes under CUDA-graph replay: C1 and C2
cd $GRAFT_REPO_ROOT
bash tools/gpu_cfg_variants.sh s4c "C1,C2" base pdl > gpurun_out/cfgv_s4_summary.txt 2>&1
for v in base pdl; do ONESWEEP_B200_LIB=$PWD/paper_2206_01784_b200/_lib/variants/$v.so timeout 300 python tools/size_sweep.py > gpurun_out/sizes_s4_$v.txt 2>&1; done
echo done
