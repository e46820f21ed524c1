for r in 1 2; do for v in E0 E1; do for w in C1 C2 C3b; do for lp in lsu tex split tex-split; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload $w --line-path $lp --no-cpu --no-e2e --no-extras --steps 8 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$w', '$lp', round(d['value'],2), d['parity_sample']['mismatches'])"
done; done; done; done
