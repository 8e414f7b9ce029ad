mkdir -p gpurun_out/p3
python tests/diag_parity.py > gpurun_out/p3/diag_3.txt 2>&1
CG_TF32_TERMS=4 python tests/diag_parity.py > gpurun_out/p3/diag_4.txt 2>&1
python tests/bench_gemm.py dgrad1:1pre fwd0:1pre wgrad1:1 > gpurun_out/p3/gemm_3.txt 2>&1
CG_TF32_TERMS=4 python tests/bench_gemm.py dgrad1:1pre fwd0:1pre wgrad1:1 > gpurun_out/p3/gemm_4.txt 2>&1
