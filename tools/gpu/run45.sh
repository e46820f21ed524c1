# Fixed-config timings of the runtime plane_levels kernels (vs the compile-time A/B builds of run43).
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r45.log
for spec in "C1 tex 2" "C3b tex 2" "C3b tex-select 2" "C3a tex-select 2" "C2 tex 4"; do
  set -- $spec
  for pu in 0 2 3 4; do
    timeout 300 python bench.py --workload $1 --line-path $2 --queries-per-lane $3 --threads 1024 --plane-levels $pu --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 tiles $3 planes $pu ->', round(d['value'],2), d['kernel']['plane_levels'], d['parity_sample']['mismatches'])" >> $O/r45.log
  done
done
cat $O/r45.log
