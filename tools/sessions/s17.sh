# device-side pass skipping: C2 (no trivial place), C3/C4 configs, small-range keys
cd $GRAFT_REPO_ROOT
bash tools/gpu_ab.sh s17 3 head route
bash tools/gpu_cfg_variants.sh s17c "C1,C3,C4" head route > gpurun_out/cfgv_s17_summary.txt 2>&1
cat gpurun_out/cfgv_s17_summary.txt
