set -u
OUT=gpurun_out/${1:-hx}; mkdir -p $OUT
for c in 1 64 256 1024; do CG_H2D_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$c.json 2>> $OUT/bench.err; done
