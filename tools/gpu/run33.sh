# PBSEQ passes unrolled (libPBU) vs a loop (default); tuned line path and tiles.
cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="lpm6cu PBU" WLS="C2 C1 C3a C3b" bash tools/ab_bench.sh > $O/r33_ab.log 2>&1
