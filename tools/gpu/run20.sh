# XOR fan-out of Phase B keys/nodes (default build) vs indexed shuffles (libXF0): parity + A/B.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "not every_chunk" > $O/r20_pytest.log 2>&1; echo "pytest rc $?" >> $O/r20_pytest.log
VARIANTS="lpm6cu XF0" WLS="C2 C1 C3a C3b" bash tools/ab_bench.sh > $O/r20_ab.log 2>&1
timeout 300 python -m pytest tests/test_gpu_store.py -m gpu -x -q -k warm > $O/r20_store_alone.log 2>&1; echo "rc $?" >> $O/r20_store_alone.log
timeout 300 python tools/store_cold.py C1 > $O/r20_store_cold.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_store.py -m gpu -x -q -k "not every_chunk" > $O/r20_store_after_parity.log 2>&1; echo "rc $?" >> $O/r20_store_after_parity.log
