set -x
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
python tests/bench_gemm.py > $O/gemm_fast.txt 2>&1
CG_GEMM_EGROUPS=1 python tests/bench_gemm.py > $O/gemm_fast_g1.txt 2>&1
CG_GEMM_GENERIC_EPI=1 python tests/bench_gemm.py > $O/gemm_generic.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench.json 2> $O/bench.err
CG_GEMM_GENERIC_EPI=1 timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench_generic.json 2> $O/bench_generic.err
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench2.json 2> $O/bench2.err
timeout 1200 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -x > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
