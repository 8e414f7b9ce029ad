set -u
OUT=gpurun_out/${1:-ix}; mkdir -p $OUT
timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "upload or copy_rows" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
grep -q "rc=0" $OUT/pytest_k.log || exit 0
for c in 0 8 16 32 64; do CG_UPLOAD_CTAS=$c timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$c.json 2>> $OUT/bench.err; done
