cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="VB3 VB2 VS0T" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r9_ab.log 2>&1
