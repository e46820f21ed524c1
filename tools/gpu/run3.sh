# Round-2 measurement pass: GPU tests (incl. slow), the default bench line (C2),
# the reference arm, launch list + one full ncu capture of the bench kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out
nproc > $O/r3_host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/r3_host.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rs > $O/r3_pytest.log 2>&1; echo "pytest rc $?" >> $O/r3_pytest.log
timeout 900 python bench.py > $O/r3_bench_c2.json 2> $O/r3_bench_c2.err; echo "bench rc $?" >> $O/r3_bench_c2.err
timeout 900 python bench.py --impl reference > $O/r3_ref_c2.json 2> $O/r3_ref_c2.err
LP=$(python -c "import json;d=json.loads(open('$O/r3_bench_c2.json').read().strip().splitlines()[-1]);print({0:'lsu',1:'tex',2:'split',3:'tex-split'}[d['kernel']['line_path']])")
echo "line path $LP" > $O/r3_lp.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r3_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r3_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r02_c2 python bench.py --line-path $LP --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r3_ncu_full.log 2>&1
python tools/ncu_summary.py $O/prof_r02_c2.ncu-rep 1073741824 > $O/r3_ncu_c2_summary.txt 2>&1
ncu -i $O/prof_r02_c2.ncu-rep --page details --csv > $O/r3_ncu_details_c2.csv 2>/dev/null
ncu -i $O/prof_r02_c2.ncu-rep --page raw --csv > $O/r3_ncu_raw_c2.csv 2>/dev/null
rm -f $O/prof_r02_c2.ncu-rep.tmp
