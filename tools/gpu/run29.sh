# Final round-2 measurement pass (after v16/v17): GPU tests (all), smoke, every workload's
# bench line (ours + reference arm), the default command's launch list, ncu --set full of
# the C2 (default), C1 and C3b bench kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > $O/r29_pytest.log 2>&1; echo "pytest rc $?" >> $O/r29_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r29_smoke.log 2>&1; echo "smoke rc $?" >> $O/r29_smoke.log
timeout 900 python bench.py > $O/r29_bench_C2.json 2> $O/r29_bench_C2.err
timeout 900 python bench.py --impl reference > $O/r29_ref_C2.json 2> $O/r29_ref_C2.err
for w in C0 C1 C3a C3b C4; do
  timeout 900 python bench.py --workload $w > $O/r29_bench_$w.json 2> $O/r29_bench_$w.err
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $O/r29_ref_$w.json 2> $O/r29_ref_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r29_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r29_ncu_launch.log 2>&1
for w in C2 C1 C3b; do
  N=$(python -c "print({'C1':268435456,'C3b':268435456,'C2':1073741824}['$w'])")
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r29_$w python bench.py --workload $w --line-path tex --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r29_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/prof_r29_$w.ncu-rep $N > $O/r29_ncu_${w}_summary.txt 2>&1
  ncu -i $O/prof_r29_$w.ncu-rep --page raw --csv > $O/r29_ncu_raw_$w.csv 2>/dev/null
  ncu -i $O/prof_r29_$w.ncu-rep --page details --csv > $O/r29_ncu_details_$w.csv 2>/dev/null
  rm -f $O/prof_r29_$w.ncu-rep
done
