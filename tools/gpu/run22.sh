# C1 / C3b with level 3 read from L2 by lane groups (smem_levels 3) on every line path,
# internal texture lines as lane quarters (default) and as sector halves (libIS1).
cd $GRAFT_REPO_ROOT
O=gpurun_out
for lib in lpm6cu IS1; do for w in C1 C3b; do for lp in lsu tex split tex-split; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$lib.so timeout 300 python bench.py --workload $w --smem-levels 3 --line-path $lp \
    --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
d=json.loads(t[-1]) if t else {}
print('$lib', '$w', 'T3', '$lp', round(d.get('value',0),2), d.get('parity_sample',{}).get('mismatches'))" >> $O/r22_t3.log
done; done; done
for i in 1 2 3 4 5 6; do LPM6CU_TRACE_BUILD=1 timeout 300 python -m pytest tests/test_gpu_store.py -m gpu -q -s -k warm >> $O/r22_store_trace.log 2>&1; done
LPM6CU_TRACE_BUILD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_store.py -m gpu -q -s -k "not every_chunk" > $O/r22_store_after_parity.log 2>&1; echo "rc $?" >> $O/r22_store_after_parity.log
