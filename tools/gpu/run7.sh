cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in VB VS0; do
LPM6CU_LIB=paper_2604_14650_b200/lib/lib$v.so timeout 900 ncu --set full --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_c1_lp1_$v python bench.py --workload C1 --line-path tex --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r7_ncu_$v.log 2>&1
python tools/ncu_summary.py $O/prof_c1_lp1_$v.ncu-rep 268435456 > $O/r7_sum_$v.txt 2>&1
ncu -i $O/prof_c1_lp1_$v.ncu-rep --page raw --csv > $O/r7_raw_$v.csv 2>/dev/null
rm -f $O/prof_c1_lp1_$v.ncu-rep
done
