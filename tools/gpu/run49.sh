# (switch not kept in the sources) A/B on C2: a quarter of the level-4 lines through the LSU (libTQ, LPM6_TEXL_QUARTER=1) with
# and without split planes, against the product library (all level-4 lines on the texture pipe).
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r49.log
for r in 1 2; do for v in lpm6cu TQ; do for pu in 0 2 4; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload C2 --line-path tex --queries-per-lane 4 --threads 1024 --plane-levels $pu --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v planes $pu ->', round(d['value'],2), d['kernel']['plane_levels'], d['parity_sample']['mismatches'])" >> $O/r49.log
done; done; done
cat $O/r49.log
