set -u
OUT=gpurun_out/${1:-sx}; mkdir -p $OUT
CG_SPMM_ASYNC_MINF=1 timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "spmm" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
grep -q "rc=0" $OUT/pytest_k.log || exit 0
for m in 129 1 65; do CG_SPMM_ASYNC_MINF=$m timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$m.json 2>> $OUT/bench.err; done
