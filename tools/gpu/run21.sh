cd $GRAFT_REPO_ROOT
O=gpurun_out
for a in plain init plain init; do timeout 300 python tools/store_warm_probe.py $a >> $O/r21_probe.log 2>&1; done
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/store_warm_probe.py eager >> $O/r21_probe.log 2>&1
timeout 300 python -m pytest tests/test_gpu_store.py -m gpu -q -k warm > $O/r21_store_alone.log 2>&1
CUDA_MODULE_LOADING=EAGER timeout 300 python -m pytest tests/test_gpu_store.py -m gpu -q -k warm > $O/r21_store_alone_eager.log 2>&1
timeout 300 python tools/store_cold.py C1 >> $O/r21_probe.log 2>&1
