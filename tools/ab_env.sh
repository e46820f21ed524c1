# usage: VALS="0 1 2" WLS="C1 C2" VAR=LPM6_TEX_LEAF_EIGHTHS bash ab_env.sh
for r in 1 2; do for v in $VALS; do for w in $WLS; do
  env $VAR=$v timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$v', d['config']['workload'], round(d['value'],2), d['parity_sample']['mismatches'])"
done; done; done
