cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line_path.py -m gpu -x -q -k "half or c2 or golden_large or line_path or tuner" > $O/r18_pytest.log 2>&1; echo "pytest rc $?" >> $O/r18_pytest.log
VARIANTS="HPIPE HNP" WLS="C2" bash tools/ab_bench.sh > $O/r18_ab.log 2>&1
for lp in tex split; do LP=$lp VARIANTS="HPIPE HNP" WLS="C2" bash tools/ab_bench.sh; done >> $O/r18_ab.log 2>&1
