# Phase B one tile at a time with 2, 3 or 4 tiles per warp through Phase A
# (queries_per_lane 2-4 at 1024 threads), texture line path; parity on the bench sample.
cd $GRAFT_REPO_ROOT
O=gpurun_out
for r in 1 2; do for w in C2 C1 C3b C3a; do for qpl in 2 3 4; do
  timeout 300 python bench.py --workload $w --line-path tex --queries-per-lane $qpl --threads 1024 \
    --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>$O/r31_err.txt | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
if not t: print('$w qpl $qpl FAILED', open('$O/r31_err.txt').read()[-400:].replace(chr(10),' ')); sys.exit()
d=json.loads(t[-1]); print('$w', 'qpl', $qpl, round(d['value'],2), d['kernel'], d['parity_sample']['mismatches'])" >> $O/r31_ab.log
done; done; done
