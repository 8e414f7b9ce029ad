set -x
O=gpurun_out/r2h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
for eg in 2 1; do CG_GEMM_EGROUPS=$eg python tests/bench_gemm.py fwd0:1pre dgrad2:1pre > $O/gemm_g$eg.txt 2>&1; done
CG_GEMM_GENERIC_EPI=1 python tests/bench_gemm.py fwd0:1pre dgrad2:1pre > $O/gemm_generic.txt 2>&1
CASES="fwd0:1pre dgrad2:1pre" bash scripts/gemm_prof.sh r2h/gemm
