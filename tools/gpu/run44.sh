# Split-plane Phase A as a product option (lpm6cu_kernel_config.plane_levels, picked by the
# tuner): the GPU tests that cover it, then every workload's bench line with the tuner.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 python -m pytest tests/test_gpu_line_path.py tests/test_gpu_stress.py tests/test_gpu_store.py tests/test_gpu_parity.py -m gpu -q -x -k "not c4_every_chunk" > $O/r44_pytest.log 2>&1; echo "pytest rc $?" >> $O/r44_pytest.log
tail -5 $O/r44_pytest.log
for w in C1 C3b C3a C2; do
  timeout 600 python bench.py --workload $w --no-cpu --no-e2e --no-extras > $O/r44_bench_$w.json 2> $O/r44_bench_$w.err
  python - <<PY
import json
t=open("$O/r44_bench_$w.json").read().strip().splitlines()
if not t: print("$w FAILED", open("$O/r44_bench_$w.err").read()[-400:])
else:
    d=json.loads(t[-1]); print("$w", round(d["value"],2), d["kernel"], d["parity_sample"])
PY
done
