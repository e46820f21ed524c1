# A/B timing of library variants on one box: VARIANTS="A B" WLS="C1 C2" bash tools/ab_bench.sh
# (paper_2604_14650_b200/lib/lib<V>.so for each variant V; two rounds, interleaved)
for r in 1 2; do for v in ${VARIANTS:-A B}; do for w in ${WLS:-C1}; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-extras \
    --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['config']['workload'], round(d['value'],2), d['parity_sample']['mismatches'])"
done; done; done
