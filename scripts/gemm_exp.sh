set -u
OUT=gpurun_out/${1:-g2}; mkdir -p $OUT
# guard against hangs: every step has its own short timeout
timeout 120 python tests/bench_gemm.py dgrad2:1pre > $OUT/quick_mask.txt 2>&1 || { echo "mask GEMM failed/hung rc=$?" >> $OUT/quick_mask.txt; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
[ -n "${NO_GEMM_BENCH:-}" ] || timeout 300 python tests/bench_gemm.py > $OUT/bench_gemm.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/launches_bench.log" 2>&1
python tests/launch_breakdown.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
for c in ${CASES:-}; do
  n=${c/:/_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 2 -c 1 \
    -o $OUT/prof_$n python tests/bench_gemm.py $c > $OUT/prof_$n.log 2>&1
done
