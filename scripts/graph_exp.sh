set -u
OUT=gpurun_out/${1:-gx}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_graphs.py -x -q > $OUT/pytest_g.log 2>&1; echo "rc=$?" >> $OUT/pytest_g.log
grep -q "rc=0" $OUT/pytest_g.log || exit 0
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for v in 0 1; do CG_GRAPHS=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$v.json 2>> $OUT/bench.err; done
