# Per-instruction attribution of the C2 and C1 bench kernels' L1 wavefronts (ncu source page):
# which SASS instructions the "global" LSU wavefronts (0.50 / 0.35 per query) belong to.
cd $GRAFT_REPO_ROOT
O=gpurun_out
for spec in "C2 4" "C1 2"; do
  set -- $spec; w=$1; q=$2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r38_$w python bench.py --workload $w --line-path tex --queries-per-lane $q --threads 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r38_ncu_$w.log 2>&1
  ncu -i $O/prof_r38_$w.ncu-rep --page source --csv > $O/r38_ncu_source_$w.csv 2>/dev/null
  ncu -i $O/prof_r38_$w.ncu-rep --page raw --csv > $O/r38_ncu_raw_$w.csv 2>/dev/null
  ls -la $O/prof_r38_$w.ncu-rep
  rm -f $O/prof_r38_$w.ncu-rep
done
