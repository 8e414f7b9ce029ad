O=gpurun_out/r3f
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $O/bench_c4.json 2> $O/bench_c4.err
CG_WGRAD_TILES_PER_SM=2 timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $O/bench_c4_t2.json 2> $O/bench_c4_t2.err
timeout 1200 python -m pytest tests/test_gpu_train_parity.py -q -x > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
