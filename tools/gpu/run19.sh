# Session re-entry measurement pass: GPU tests, every workload's line (ours + reference arm),
# launch list of the default command.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=10 > $O/r19_pytest.log 2>&1; echo "pytest rc $?" >> $O/r19_pytest.log
timeout 900 python bench.py > $O/r19_bench_C2.json 2> $O/r19_bench_C2.err
timeout 900 python bench.py --impl reference > $O/r19_ref_C2.json 2> $O/r19_ref_C2.err
for w in C0 C1 C3a C3b C4; do
  timeout 900 python bench.py --workload $w > $O/r19_bench_$w.json 2> $O/r19_bench_$w.err
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $O/r19_ref_$w.json 2> $O/r19_ref_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r19_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r19_ncu_launch.log 2>&1
