# Deep-level offload (LookupParams::l2_share, env LPM6CU_L2_SHARE): share of tiles whose
# deepest staged level is read from L2 by lane groups. Parity checked on the bench sample.
cd $GRAFT_REPO_ROOT
O=gpurun_out
LPM6CU_TRACE_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_store.py -m gpu -q -s -k "not every_chunk" > $O/r23_store_after_parity.log 2>&1; echo "rc $?" >> $O/r23_store_after_parity.log
timeout 1500 python -m pytest tests -m gpu -q -k "not every_chunk" > $O/r23_pytest.log 2>&1; echo "pytest rc $?" >> $O/r23_pytest.log
for r in 1 2; do for w in C1 C3b C2; do for lp in tex tex-split; do for sh in 0 2 3 4 5; do
  LPM6CU_L2_SHARE=$sh timeout 300 python bench.py --workload $w --line-path $lp \
    --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
d=json.loads(t[-1]) if t else {}
print('$w', '$lp', 'share', $sh, round(d.get('value',0),2), d.get('parity_sample',{}).get('mismatches'))" >> $O/r23_share.log
done; done; done; done
