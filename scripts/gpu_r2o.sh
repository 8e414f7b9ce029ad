O=gpurun_out/r2o
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "mode3 or tcgen05" > $O/pytest_mode3.log 2>&1
echo "rc $?" >> $O/pytest_mode3.log
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench.json 2> $O/bench.err
CG_GEMM_BX=1 timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench_bx.json 2> $O/bench_bx.err
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench2.json 2> $O/bench2.err
CG_GEMM_BX=1 timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench_bx2.json 2> $O/bench_bx2.err
CG_GEMM_BX=1 timeout 1200 python -m pytest tests/test_gpu_train_parity.py -q -x > $O/pytest_parity_bx.log 2>&1
echo "rc $?" >> $O/pytest_parity_bx.log
CG_GEMM_BX=1 timeout 300 ncu --set full --clock-control none -k regex:k_gemm_tc -s 18 -c 8 -o $O/prof_gemm_bx python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-exchange > $O/prof_bx.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_gemm_tc -s 18 -c 8 -o $O/prof_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-exchange > $O/prof.log 2>&1
