cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2_pytest.log
VARIANTS="R1 R2" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > gpurun_out/r2_ab.log 2>&1
