O=gpurun_out/r2m
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench.json 2> $O/bench.err
CG_MASK_BITS=0 timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench_nobits.json 2> $O/bench_nobits.err
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench2.json 2> $O/bench2.err
for v in "" "CG_SPMM_FLAGS=0" "CG_L0_OWNER=0"; do
  env $v timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > "$O/bench_c3_${v:-default}.json" 2>> $O/c3.err
done
timeout 1500 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py tests/test_gpu_multirank.py -q > $O/pytest_parity.log 2>&1
echo "rc $?" >> $O/pytest_parity.log
