cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="VB VX" WLS="C2" bash tools/ab_bench.sh > $O/r6_ab_xchg.log 2>&1
for lp in lsu tex split; do LP=$lp VARIANTS="VB VS0 VR0" WLS="C1 C3a C3b" bash tools/ab_bench.sh; done > $O/r6_ab_lp.log 2>&1
