O=gpurun_out/r2w
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -x > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
timeout 900 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
CG_GCN_TFL=0 timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/bench_c3_agg.json 2> $O/bench_c3_agg.err
timeout 1500 python -m pytest tests/test_gpu_golden_big.py -q > $O/pytest_big.log 2>&1
echo "rc $?" >> $O/pytest_big.log
