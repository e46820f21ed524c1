# Re-entry check of the PBSEQ kernel (after run33): GPU tests (all), smoke, the default
# bench line + reference arm, the launch list of the default command, ncu --set full of
# the C2 bench kernel as the tuner runs it.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > $O/r34_pytest.log 2>&1; echo "pytest rc $?" >> $O/r34_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r34_smoke.log 2>&1; echo "smoke rc $?" >> $O/r34_smoke.log
timeout 900 python bench.py > $O/r34_bench_C2.json 2> $O/r34_bench_C2.err
timeout 900 python bench.py --impl reference > $O/r34_ref_C2.json 2> $O/r34_ref_C2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r34_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r34_ncu_launch.log 2>&1
for w in C2; do
  N=1073741824
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r34_$w python bench.py --workload $w --line-path tex --queries-per-lane 4 --threads 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r34_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/prof_r34_$w.ncu-rep $N > $O/r34_ncu_${w}_summary.txt 2>&1
  ncu -i $O/prof_r34_$w.ncu-rep --page raw --csv > $O/r34_ncu_raw_$w.csv 2>/dev/null
  ncu -i $O/prof_r34_$w.ncu-rep --page details --csv > $O/r34_ncu_details_$w.csv 2>/dev/null
  ncu -i $O/prof_r34_$w.ncu-rep --page source --csv > $O/r34_ncu_source_$w.csv 2>/dev/null
  rm -f $O/prof_r34_$w.ncu-rep
done
