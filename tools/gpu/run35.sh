# Measurement pass on the PBSEQ kernel (v18/v19): every workload's bench line (ours +
# reference arm), ncu --set full of the C1 and C3b bench kernels as the tuner runs them
# (texture line path 1, 2 tiles per warp); the C2 capture and the launch list are run34's.
cd $GRAFT_REPO_ROOT
O=gpurun_out
for w in C0 C1 C3a C3b C4; do
  timeout 900 python bench.py --workload $w > $O/r35_bench_$w.json 2> $O/r35_bench_$w.err
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $O/r35_ref_$w.json 2> $O/r35_ref_$w.err
done
for w in C1 C3b; do
  N=268435456
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r35_$w python bench.py --workload $w --line-path tex --queries-per-lane 2 --threads 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r35_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/prof_r35_$w.ncu-rep $N > $O/r35_ncu_${w}_summary.txt 2>&1
  ncu -i $O/prof_r35_$w.ncu-rep --page raw --csv > $O/r35_ncu_raw_$w.csv 2>/dev/null
  ncu -i $O/prof_r35_$w.ncu-rep --page details --csv > $O/r35_ncu_details_$w.csv 2>/dev/null
  rm -f $O/prof_r35_$w.ncu-rep
done
