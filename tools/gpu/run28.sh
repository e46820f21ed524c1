# Leaf-image kernels: addresses two tiles ahead (default) vs one (libPF1), C0.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c0 or leaf or golden" > $O/r28_pytest.log 2>&1; echo "pytest rc $?" >> $O/r28_pytest.log
for r in 1 2 3; do for v in lpm6cu PF1; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload C0 --no-cpu --no-e2e --no-extras --steps 50 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],2), round(d['ms_per_step']*1e3,2), 'us', d['parity_sample']['mismatches'])" >> $O/r28_ab.log
done; done
