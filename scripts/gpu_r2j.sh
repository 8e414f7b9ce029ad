set -x
O=gpurun_out/r2j
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
for pf in 0 2 4 8 12; do CG_GEMM_PF=$pf python tests/bench_gemm.py fwd0:1pre fwd1:1pre fwd2:1pre dgrad1:1pre dgrad2:1pre wgrad2:1 wgrad1:1 wgrad0:1 > $O/gemm_pf$pf.txt 2>&1; done
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench.json 2> $O/bench.err
CG_GEMM_PF=0 timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench_pf0.json 2> $O/bench_pf0.err
