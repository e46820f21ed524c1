# Lane texel base per level (default build) vs the previous commit (libPREV).
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not every_chunk" > $O/r27_pytest.log 2>&1; echo "pytest rc $?" >> $O/r27_pytest.log
VARIANTS="lpm6cu PREV" WLS="C2 C1 C3a C3b" bash tools/ab_bench.sh > $O/r27_ab.log 2>&1
