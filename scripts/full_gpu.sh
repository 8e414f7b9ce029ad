set -u
OUT=gpurun_out/${1:-fx}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench.json 2>> $OUT/bench.err
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $OUT/bench_c4.json 2>> $OUT/bench.err
