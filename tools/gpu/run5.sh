cd $GRAFT_REPO_ROOT
O=gpurun_out
VARIANTS="VB VW0 VS0 VR0" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r5_ab.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > $O/r5_pytest.log 2>&1; echo "pytest rc $?" >> $O/r5_pytest.log
python tools/store_cold.py C1 > $O/r5_store_cold_c1.json 2>&1
python tools/store_cold.py C2 > $O/r5_store_cold_c2.json 2>&1
