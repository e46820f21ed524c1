cd $GRAFT_REPO_ROOT
O=gpurun_out
for lp in tex split; do LP=$lp VARIANTS="H0 HIS" WLS="C2" bash tools/ab_bench.sh; done > $O/r17_ab.log 2>&1
