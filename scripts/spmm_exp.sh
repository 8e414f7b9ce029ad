set -u
OUT=gpurun_out/${1:-sx}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "spmm" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$i.json 2>> $OUT/bench.err; done
