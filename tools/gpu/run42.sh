# A/B: split-plane Phase A (libPL, LPM6_PLANES=1: LDS.32 probes of the high words, low
# words only when a lane of the warp ties; tools/hilo_sim.py is the host model) vs the
# packed 8-byte probes. Parity of the variant first (golden fixtures, every workload's
# sample through bench.py's parity_sample), then timing.
cd $GRAFT_REPO_ROOT
O=gpurun_out
LPM6CU_LIB=paper_2604_14650_b200/lib/libPL.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_line_path.py -m gpu -q -x -k "not c4_every_chunk" > $O/r42_pytest_PL.log 2>&1; echo "rc $?" >> $O/r42_pytest_PL.log
tail -4 $O/r42_pytest_PL.log
VARIANTS="lpm6cu PL" WLS="C1 C2 C3a C3b" bash tools/ab_bench.sh > $O/r42_ab.log 2>&1
cat $O/r42_ab.log
