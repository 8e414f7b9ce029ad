set -u
OUT=gpurun_out/${1:-sp}; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 24 -c 8 \
  -o "$OUT/prof_spmm" python bench.py --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/prof_spmm.log" 2>&1
CG_SPMM_ASYNC=1 timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "spmm" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
for v in 1 0; do CG_SPMM_G4=$v CG_SPMM_ASYNC=1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_g4_$v.json 2>> $OUT/bench.err; done
