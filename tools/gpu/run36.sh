# Re-entry validation (session 5 of round 2): GPU tests, smoke, the default bench line
# and the reference arm on the restored checkpoint.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > $O/r36_pytest.log 2>&1; echo "pytest rc $?" >> $O/r36_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r36_smoke.log 2>&1; echo "smoke rc $?" >> $O/r36_smoke.log
timeout 900 python bench.py > $O/r36_bench_C2.json 2> $O/r36_bench_C2.err
timeout 900 python bench.py --impl reference > $O/r36_ref_C2.json 2> $O/r36_ref_C2.err
tail -3 $O/r36_pytest.log; tail -2 $O/r36_smoke.log; head -c 600 $O/r36_bench_C2.json
