# Compile-time plane levels (PLANES = 2, 3, all): the GPU tests that cover them, fixed-config
# timings, then every workload's tuned bench line.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests/test_gpu_line_path.py tests/test_gpu_stress.py tests/test_gpu_store.py -m gpu -q -x > $O/r46_pytest.log 2>&1; echo "pytest rc $?" >> $O/r46_pytest.log
tail -5 $O/r46_pytest.log
: > $O/r46.log
for spec in "C1 tex 2" "C3b tex 2" "C3b tex-select 2"; do
  set -- $spec
  for pu in 0 2 3 4; do
    timeout 300 python bench.py --workload $1 --line-path $2 --queries-per-lane $3 --threads 1024 --plane-levels $pu --no-cpu --no-e2e --no-extras --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2 tiles $3 planes $pu ->', round(d['value'],2), d['kernel']['plane_levels'], d['parity_sample']['mismatches'])" >> $O/r46.log
  done
done
cat $O/r46.log
for w in C1 C3b C3a C2; do
  timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-extras > $O/r46_bench_$w.json 2> $O/r46_bench_$w.err
  python - <<PY
import json
t=open("$O/r46_bench_$w.json").read().strip().splitlines()
if not t: print("$w FAILED", open("$O/r46_bench_$w.err").read()[-400:])
else:
    d=json.loads(t[-1]); k=d["kernel"]; print("$w tuned", round(d["value"],2), "lp", k["line_path"], "tiles", k["queries_per_lane"], "planes", k["plane_levels"], d["parity_sample"]["mismatches"])
PY
done
