# Static staged-level count (default build) vs runtime (libTA0): A/B on every single-FIB workload + parity.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not every_chunk" > $O/r25_pytest.log 2>&1; echo "pytest rc $?" >> $O/r25_pytest.log
VARIANTS="lpm6cu TA0" WLS="C2 C1 C3a C3b" bash tools/ab_bench.sh > $O/r25_ab.log 2>&1
