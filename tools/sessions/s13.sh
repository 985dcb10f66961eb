# key prefetch depth in the ranking loop (C2)
cd $GRAFT_REPO_ROOT
bash tools/gpu_ab.sh s13 3 base pf1 pf3
