# Measurement pass with the split-plane descent in the tuner (v20): all GPU tests, smoke,
# every workload's bench line and reference arm, ncu --set full of the C1 and C3b bench
# kernels as the tuner now runs them, the launch list of the default command.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=8 > $O/r47_pytest.log 2>&1; echo "pytest rc $?" >> $O/r47_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r47_smoke.log 2>&1; echo "smoke rc $?" >> $O/r47_smoke.log
for w in C2 C1 C3a C3b C4 C0; do
  timeout 900 python bench.py --workload $w > $O/r47_bench_$w.json 2> $O/r47_bench_$w.err
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $O/r47_ref_$w.json 2> $O/r47_ref_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r47_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r47_ncu_launch.log 2>&1
for w in C1 C3b; do
  N=268435456
  # the tuned config of this workload from its bench line
  read LP QPL PU <<< $(python -c "
import json; d=json.loads(open('$O/r47_bench_$w.json').read().strip().splitlines()[-1])['kernel']
print({0:'lsu',1:'tex',2:'split',3:'tex-split',4:'tex-select'}[d['line_path']], d['queries_per_lane'], d['plane_levels'])")
  echo "$w: line path $LP tiles $QPL planes $PU" > $O/r47_ncu_${w}_config.txt
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r47_$w python bench.py --workload $w --line-path $LP --queries-per-lane $QPL --plane-levels $PU --threads 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r47_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/prof_r47_$w.ncu-rep $N > $O/r47_ncu_${w}_summary.txt 2>&1
  ncu -i $O/prof_r47_$w.ncu-rep --page raw --csv > $O/r47_ncu_raw_$w.csv 2>/dev/null
  ncu -i $O/prof_r47_$w.ncu-rep --page details --csv > $O/r47_ncu_details_$w.csv 2>/dev/null
  ncu -i $O/prof_r47_$w.ncu-rep --page source --csv > $O/r47_ncu_source_$w.csv 2>/dev/null
  rm -f $O/prof_r47_$w.ncu-rep
done
tail -3 $O/r47_pytest.log; tail -1 $O/r47_smoke.log
