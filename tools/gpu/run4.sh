cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > $O/r4_pytest.log 2>&1; echo "pytest rc $?" >> $O/r4_pytest.log
python tools/store_cold.py C1 > $O/r4_store_cold_c1.json 2>&1
python tools/store_cold.py C2 > $O/r4_store_cold_c2.json 2>&1
CUDA_MODULE_LOADING=EAGER python tools/store_cold.py C1 > $O/r4_store_cold_c1_eager.json 2>&1
./tools/latency_abi > $O/r4_latency_abi.json 2>&1
for r in 1 2; do for v in R1 R2; do for lp in lsu tex split tex-split; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload C1 --line-path $lp --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'C1', '$lp', round(d['value'],2), d['parity_sample']['mismatches'])"
done; done; done > $O/r4_ab_c1.log 2>&1
