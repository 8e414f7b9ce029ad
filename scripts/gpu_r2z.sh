O=gpurun_out/r2z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
python tests/bench_gemm.py wgrad2:1 wgrad1:1 wgrad0:1 > $O/gemm_wgrad.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-exchange > $O/bench$i.json 2> $O/bench$i.err; done
timeout 1500 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -x > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
