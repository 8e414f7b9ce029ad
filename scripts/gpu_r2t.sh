O=gpurun_out/r2t
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -x > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-exchange > $O/bench$i.json 2> $O/bench$i.err
CG_GCN_TFL=0 timeout 600 python bench.py --no-cpu-baseline --no-exchange > $O/bench_agg$i.json 2> $O/bench_agg$i.err
done
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 1500 python -m pytest tests/test_gpu_golden_big.py -q > $O/pytest_big.log 2>&1
echo "rc $?" >> $O/pytest_big.log
