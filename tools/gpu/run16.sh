cd $GRAFT_REPO_ROOT
O=gpurun_out
w=C2; N=1073741824
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r02h_$w python bench.py --workload $w --line-path tex --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r16_ncu_$w.log 2>&1
python tools/ncu_summary.py $O/prof_r02h_$w.ncu-rep $N > $O/r16_ncu_${w}_summary.txt 2>&1
ncu -i $O/prof_r02h_$w.ncu-rep --page raw --csv > $O/r16_ncu_raw_$w.csv 2>/dev/null
ncu -i $O/prof_r02h_$w.ncu-rep --page details --csv > $O/r16_ncu_details_$w.csv 2>/dev/null
ncu -i $O/prof_r02h_$w.ncu-rep --page source --csv --print-source sass > $O/r16_ncu_source_$w.csv 2>/dev/null
rm -f $O/prof_r02h_$w.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r16_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r16_ncu_launch.log 2>&1
