cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r1_pytest.log
VARIANTS="R0 R1" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > gpurun_out/r1_ab.log 2>&1
