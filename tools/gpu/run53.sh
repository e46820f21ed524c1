# Final check after the common.hpp rewrite: all GPU tests, smoke, the default bench line, the reference arm,
# and the randomised every-mode parity stress under four fresh seeds x 200 FIBs.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/r53_pytest.log 2>&1; echo "pytest rc $?" >> $O/r53_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r53_smoke.log 2>&1; echo "smoke rc $?" >> $O/r53_smoke.log
timeout 900 python bench.py > $O/r53_bench_C2.json 2> $O/r53_bench_C2.err
timeout 900 python bench.py --impl reference > $O/r53_ref_C2.json 2> $O/r53_ref_C2.err
: > $O/r53_soak.log
for seed in 11 12 13 14; do
  LPM6_STRESS_SEED=$seed LPM6_STRESS_ITERS=200 timeout 1500 python -m pytest tests/test_gpu_stress.py -m gpu -q >> $O/r53_soak.log 2>&1
  echo "seed $seed rc $?" >> $O/r53_soak.log
done
tail -3 $O/r53_pytest.log; tail -2 $O/r53_smoke.log; grep "rc " $O/r53_soak.log
python - <<'PY'
import json
for f in ("r53_bench_C2","r53_ref_C2"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["value"],3), d.get("e2e",{}) and round(d["e2e"]["value"],3), d.get("clocks"))
PY
