# Last check of the committed tree (0d7b1c9): all GPU tests, smoke, default bench line, reference arm, C1.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/r55_pytest.log 2>&1; echo "pytest rc $?" >> $O/r55_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r55_smoke.log 2>&1; echo "smoke rc $?" >> $O/r55_smoke.log
timeout 900 python bench.py > $O/r55_bench_C2.json 2> $O/r55_bench_C2.err
timeout 900 python bench.py --impl reference > $O/r55_ref_C2.json 2> $O/r55_ref_C2.err
timeout 900 python bench.py --workload C1 --no-cpu > $O/r55_bench_C1.json 2> $O/r55_bench_C1.err
tail -3 $O/r55_pytest.log; tail -2 $O/r55_smoke.log
python - <<'PY'
import json
for f in ("r55_bench_C2","r55_ref_C2","r55_bench_C1"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["value"],3), d.get("kernel"), d.get("e2e",{}) and round(d["e2e"]["value"],3), d.get("extras",{}).get("store_commit") if isinstance(d.get("extras"),dict) else None)
PY
