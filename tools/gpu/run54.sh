# Evidence refresh on the final tree: launch list of the default command and one ncu --set full
# capture of the C2 bench kernel as the tuner runs it (after the plain bench run exited 0 in run53).
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r54_bench_C2_short.json 2> $O/r54_bench_C2_short.err; echo "bench rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r54_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r54_ncu_launch.log 2>&1; echo "launch list rc $?"
w=C2; N=1073741824
read LP QPL PU <<< $(python -c "
import json; d=json.loads(open('$O/r54_bench_C2_short.json').read().strip().splitlines()[-1])['kernel']
print({0:'lsu',1:'tex',2:'split',3:'tex-split',4:'tex-select'}[d['line_path']], d['queries_per_lane'], d['plane_levels'])")
echo "$w: line path $LP tiles $QPL planes $PU" > $O/r54_ncu_${w}_config.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r54_$w python bench.py --workload $w --line-path $LP --queries-per-lane $QPL --plane-levels $PU --threads 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r54_ncu_$w.log 2>&1; echo "ncu rc $?"
python tools/ncu_summary.py $O/prof_r54_$w.ncu-rep $N > $O/r54_ncu_${w}_summary.txt 2>&1
ncu -i $O/prof_r54_$w.ncu-rep --page details --csv > $O/r54_ncu_details_$w.csv 2>/dev/null
ncu -i $O/prof_r54_$w.ncu-rep --page source --csv > $O/r54_ncu_source_$w.csv 2>/dev/null
rm -f $O/prof_r54_$w.ncu-rep
cat $O/r54_ncu_${w}_config.txt; cat $O/r54_ncu_${w}_summary.txt | head -30
