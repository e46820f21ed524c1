cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=8 > $O/r15_pytest.log 2>&1; echo "pytest rc $?" >> $O/r15_pytest.log
timeout 900 python bench.py > $O/r15_bench_c2.json 2> $O/r15_bench_c2.err
timeout 900 python bench.py --workload C4 > $O/r15_bench_C4.json 2> $O/r15_bench_C4.err
