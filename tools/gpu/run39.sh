# (code: commit 0d11088) A/B: Phase B's query keys loaded by every lane of the group from the address stream
# (libGKL1: at the start of each pass; libGKL2: one pass ahead) vs broadcast by shuffles.
cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="lpm6cu GKL1 GKL2" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r39_ab.log 2>&1
cat $O/r39_ab.log
