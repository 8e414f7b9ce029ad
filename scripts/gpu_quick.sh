#!/usr/bin/env bash
# Quick GPU iteration: parity tests, one bench line, the launch list.
set -u
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 600 python tests/diag_tf32_rounding.py > "$OUT/diag.log" 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} \
  > "$OUT/launches_bench.log" 2>&1
python tests/launch_breakdown.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
if [ -n "${PROF_K:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$PROF_K" -s ${PROF_S:-15} -c ${PROF_C:-5} \
    -o "$OUT/prof_${PROF_NAME:-k}" python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} \
    > "$OUT/prof.log" 2>&1
fi
echo done > "$OUT/DONE"
