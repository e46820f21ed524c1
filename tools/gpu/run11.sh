cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_line_path.py tests/test_gpu_stress.py tests/test_gpu_properties.py -m gpu -x -q > $O/r11_pytest.log 2>&1; echo "pytest rc $?" >> $O/r11_pytest.log
VARIANTS="LP4" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r11_ab.log 2>&1
LP=tex-select VARIANTS="LP4" WLS="C1 C3a C3b" bash tools/ab_bench.sh >> $O/r11_ab.log 2>&1
