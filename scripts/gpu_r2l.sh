O=gpurun_out/r2l
mkdir -p $O
python tests/bench_spmm.py 2449029 26.25 48 100 256 > $O/spmm_c4_new.txt 2>&1
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 1200 ncu --set full --clock-control none -k regex:k_spmm -s 20 -c 5 -o $O/prof_spmm_c4 python bench.py --config c4 --steps 1 --warmup 4 --no-cpu-baseline > $O/prof_spmm_c4.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_golden_big.py tests/test_gpu_kernels.py -q > $O/pytest_big.log 2>&1
echo "rc $?" >> $O/pytest_big.log
