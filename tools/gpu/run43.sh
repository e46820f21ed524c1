# A/B: split-plane Phase A on levels 1-2 only (libPL3: level 3 packed, its high words tie
# too often) and on level 1 only (libPL2), next to every staged level (libPL) and the
# packed probes; parity of libPL3 first.
cd $GRAFT_REPO_ROOT
O=gpurun_out
LPM6CU_LIB=paper_2604_14650_b200/lib/libPL3.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_line_path.py -m gpu -q -x -k "not c4_every_chunk" > $O/r43_pytest_PL3.log 2>&1; echo "rc $?" >> $O/r43_pytest_PL3.log
tail -4 $O/r43_pytest_PL3.log
VARIANTS="lpm6cu PL3 PL2 PL" WLS="C1 C3b C3a C2" bash tools/ab_bench.sh > $O/r43_ab.log 2>&1
cat $O/r43_ab.log
