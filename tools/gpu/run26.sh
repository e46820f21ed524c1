# Root search as a byte-offset walk (default) vs the indexed form (libRW0).
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_line_path.py -m gpu -q -x -k "not every_chunk" > $O/r26_pytest.log 2>&1; echo "pytest rc $?" >> $O/r26_pytest.log
VARIANTS="lpm6cu RW0" WLS="C2 C1 C3a C3b" bash tools/ab_bench.sh > $O/r26_ab.log 2>&1
