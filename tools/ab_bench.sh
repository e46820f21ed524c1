# A/B timing of library variants on one box: VARIANTS="A B" WLS="C1 C2" bash tools/ab_bench.sh
# (paper_2604_14650_b200/lib/lib<V>.so for each variant V; two rounds, interleaved;
# LP=lsu|tex|split|tex-split|tune, default tune). Prints variant, workload, G/s,
# the line path the run used, parity mismatches of the checked sample.
for r in 1 2; do for v in ${VARIANTS:-A B}; do for w in ${WLS:-C1}; do
  LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload $w --line-path ${LP:-tune} \
    --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/tmp/ab_err.txt | python -c "
import json,sys
t=sys.stdin.read().strip().splitlines()
if not t: print('$v', '$w', 'FAILED', open('/tmp/ab_err.txt').read()[-300:].replace(chr(10),' ')); sys.exit()
d=json.loads(t[-1]); print('$v', d['config']['workload'], round(d['value'],2), 'lp', d['kernel']['line_path'], d['parity_sample']['mismatches'])"
done; done; done
