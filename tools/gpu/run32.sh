# Tuner over line paths x tiles per warp (1, 2, 4 on the texture leaf paths): GPU tests and
# every workload's tuned bench line (no CPU baseline / e2e, for speed).
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -k "not every_chunk" > $O/r32_pytest.log 2>&1; echo "pytest rc $?" >> $O/r32_pytest.log
for w in C2 C1 C3a C3b C4 C0; do
  timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-extras > $O/r32_bench_$w.json 2> $O/r32_bench_$w.err
done
