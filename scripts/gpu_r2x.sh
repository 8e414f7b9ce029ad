O=gpurun_out/r2x
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
