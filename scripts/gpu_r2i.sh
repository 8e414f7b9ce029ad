set -x
O=gpurun_out/r2i
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
python tests/bench_gemm.py > $O/gemm_default.txt 2>&1
CG_GEMM_NO_BRES=1 python tests/bench_gemm.py fwd0:1pre fwd2:1pre dgrad2:1pre > $O/gemm_nobres.txt 2>&1
CG_GEMM_EGROUPS=2 python tests/bench_gemm.py fwd0:1pre fwd2:1pre dgrad2:1pre > $O/gemm_g2.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench.json 2> $O/bench.err
CASES="fwd0:1pre dgrad2:1pre fwd2:1pre" bash scripts/gemm_prof.sh r2i/gemm
