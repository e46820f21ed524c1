cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_line_path.py tests/test_gpu_parity.py -m gpu -x -q -k "c2 or line_path or golden or texture or tuner" > $O/r13_pytest.log 2>&1; echo "pytest rc $?" >> $O/r13_pytest.log
for lp in tune tex tex-split; do LP=$lp VARIANTS="S2 BASE" WLS="C2" bash tools/ab_bench.sh; done > $O/r13_ab.log 2>&1
VARIANTS="S2" WLS="C1 C3a C3b C4" bash tools/ab_bench.sh >> $O/r13_ab.log 2>&1
