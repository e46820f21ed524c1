# Parity soak (re-run on the v20 kernels: the stress test now covers the split-plane descent too):
# the randomised every-mode stress test (random FIBs x every shared-memory
# split x line path x tile count x checked/unchecked x address/key/search input, against
# the CPU oracle on every boundary +-1) under 10 more seeds x 200 FIBs each.
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r37_soak.log
for seed in 1 2 3 4 5 6 7 8 9 10; do
  LPM6_STRESS_SEED=$seed LPM6_STRESS_ITERS=200 timeout 1500 python -m pytest tests/test_gpu_stress.py -m gpu -q >> $O/r37_soak.log 2>&1
  echo "seed $seed rc $?" >> $O/r37_soak.log
done
grep "rc " $O/r37_soak.log
