# (switch not kept in the sources) A/B: texel addresses of C2's internal L2 level and half-line leaves from a per-level
# lane base (libTBA, LPM6_TEX_BASE_ALL=1: 64 fewer LEA in the C2 bench kernel) vs per slot.
cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="lpm6cu TBA" WLS="C2 C4" bash tools/ab_bench.sh > $O/r41_ab.log 2>&1
cat $O/r41_ab.log
