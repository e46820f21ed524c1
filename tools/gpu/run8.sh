cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_line_path.py tests/test_gpu_parity.py -m gpu -x -q -k "not every_chunk" > $O/r8_pytest.log 2>&1; echo "pytest rc $?" >> $O/r8_pytest.log
VARIANTS="VB2 VT0 VS0T" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r8_ab.log 2>&1
LP=tex VARIANTS="VB2 VT0 VS0T" WLS="C1" bash tools/ab_bench.sh > $O/r8_ab_c1tex.log 2>&1
