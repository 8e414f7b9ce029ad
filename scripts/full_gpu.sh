set -u
OUT=gpurun_out/${1:-fx}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_all.log 2>&1; echo "rc=$?" >> $OUT/pytest_all.log
for v in 1 0; do CG_PDL=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_pdl$v.json 2>> $OUT/bench.err; done
CG_PDL=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_pdl1b.json 2>> $OUT/bench.err
