# Measurement pass after the r02 kernel changes: GPU tests, default bench line (C2),
# reference arm, every workload's line, ncu captures (C1, C2, C3b), torchrun harness check.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=10 > $O/r10_pytest.log 2>&1; echo "pytest rc $?" >> $O/r10_pytest.log
timeout 900 python bench.py > $O/r10_bench_c2.json 2> $O/r10_bench_c2.err
timeout 900 python bench.py --impl reference > $O/r10_ref_c2.json 2> $O/r10_ref_c2.err
for w in C0 C1 C3a C3b C4; do
  timeout 900 python bench.py --workload $w > $O/r10_bench_$w.json 2> $O/r10_bench_$w.err
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > $O/r10_ref_$w.json 2> $O/r10_ref_$w.err
done
for w in C1 C3b C2; do
  LP=$(python -c "import json;d=json.loads(open('$O/r10_bench_$w.json' if '$w'!='C2' else '$O/r10_bench_c2.json').read().strip().splitlines()[-1]);print({0:'lsu',1:'tex',2:'split',3:'tex-split'}[d['kernel']['line_path']])")
  N=$(python -c "print({'C1':268435456,'C3b':268435456,'C2':1073741824}['$w'])")
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:lpm6_lookup_kernel --launch-skip 3 --launch-count 1 -o $O/prof_r02_$w python bench.py --workload $w --line-path $LP --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r10_ncu_$w.log 2>&1
  python tools/ncu_summary.py $O/prof_r02_$w.ncu-rep $N > $O/r10_ncu_${w}_summary.txt 2>&1
  ncu -i $O/prof_r02_$w.ncu-rep --page raw --csv > $O/r10_ncu_raw_$w.csv 2>/dev/null
  ncu -i $O/prof_r02_$w.ncu-rep --page details --csv > $O/r10_ncu_details_$w.csv 2>/dev/null
  echo "$LP" > $O/r10_lp_$w.txt
  rm -f $O/prof_r02_$w.ncu-rep
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r10_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > $O/r10_ncu_launch.log 2>&1
LPM6_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --standalone --nproc-per-node 2 bench.py --gpus 2 --steps 2 --warmup 1 --no-extras > $O/r10_torchrun2.json 2> $O/r10_torchrun2.err
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/r10_torchrun2_ref.json 2> $O/r10_torchrun2_ref.err
