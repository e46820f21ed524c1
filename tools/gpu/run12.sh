cd $GRAFT_REPO_ROOT
O=gpurun_out
for lp in lsu tex split tex-split; do LP=$lp VARIANTS="HP" WLS="C2" bash tools/ab_bench.sh; done > $O/r12b_ab.log 2>&1
