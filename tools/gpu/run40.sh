# (code: commit 2c8c686) A/B: Phase B's query keys through a per-warp shared-memory slot (libKSM: one STS.64 and
# four broadcast LDS.64 per lane and tile; node indices still shuffled) vs eight shuffles,
# on the final PBSEQ kernels (C1's image leaves room for the 8.4 KB of key slots).
cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="lpm6cu KSM" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r40_ab.log 2>&1
cat $O/r40_ab.log
