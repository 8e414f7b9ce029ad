O=gpurun_out/r2y
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -k "transform_first or graph" > $O/pytest_tfl.log 2>&1
echo "rc $?" >> $O/pytest_tfl.log
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $O/bench_c4.json 2> $O/bench_c4.err
