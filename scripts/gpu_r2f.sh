set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_train_parity.py -q -x > $O/pytest.log 2>&1
echo "rc $?" >> $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
CASES="fwd0:1pre dgrad2:1pre" bash scripts/gemm_prof.sh r2f/gemm
