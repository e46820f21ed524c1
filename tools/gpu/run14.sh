cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not every_chunk" > $O/r14_pytest.log 2>&1; echo "pytest rc $?" >> $O/r14_pytest.log
for lp in tune lsu tex split tex-split; do LP=$lp VARIANTS="HALF BASE" WLS="C2" bash tools/ab_bench.sh; done > $O/r14_ab.log 2>&1
