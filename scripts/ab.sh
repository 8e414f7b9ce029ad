set -u
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "softmax" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
timeout 600 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -x > $OUT/pytest_t.log 2>&1; echo "rc=$?" >> $OUT/pytest_t.log
for r in 1 2; do
(cd ab_head && timeout 300 python bench.py --no-cpu-baseline --steps 20 > ../$OUT/bench_head_$r.json 2>/dev/null)
timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_new_$r.json 2>/dev/null
done
