set -u
OUT=gpurun_out/${1:-cx}; mkdir -p $OUT
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $OUT/bench_c4.json 2>> $OUT/err
timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $OUT/bench_c3.json 2>> $OUT/err
