set -u
OUT=gpurun_out/${1:-fx}; mkdir -p $OUT
timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
grep -q "rc=0" $OUT/pytest_k.log || exit 0
timeout 200 python tests/bench_gemm.py fwd0:1pre fwd1:1pre fwd2:1pre dgrad1:1pre dgrad2:1pre > $OUT/gemm.txt 2>&1
for v in 1 0; do CG_MASK_BITS=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_bits$v.json 2>> $OUT/bench.err; done
