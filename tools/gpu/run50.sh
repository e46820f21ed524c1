# (the PTX form was not kept) A/B: the split-plane probe step in PTX (the library as built for this run) vs the compiler's lowering
# (libPCPP, LPM6_PLANE_PTX=0); parity of the PTX form first.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_line_path.py tests/test_gpu_stress.py -m gpu -q -x > $O/r50_pytest.log 2>&1; echo "pytest rc $?" >> $O/r50_pytest.log
tail -3 $O/r50_pytest.log
: > $O/r50.log
for r in 1 2; do for v in lpm6cu PCPP; do
  for spec in "C1 tex 2 3" "C3b tex-select 2 4" "C3b tex-select 4 4" "C1 tex 4 3"; do
    set -- $spec
    LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 300 python bench.py --workload $1 --line-path $2 --queries-per-lane $3 --threads 1024 --plane-levels $4 --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $1 $2 tiles $3 planes $4 ->', round(d['value'],2), d['kernel']['plane_levels'], d['parity_sample']['mismatches'])" >> $O/r50.log
  done
done; done
cat $O/r50.log
