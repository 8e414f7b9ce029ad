#!/usr/bin/env bash
# One gpurun call: GPU parity tests, the bench line (both arms), the launch
# list and one full ncu capture of the SpMM (and the tcgen05 GEMM).
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [tag]'
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; grep -m1 "model name" /proc/cpuinfo >> "$OUT/nproc.txt"; free -g >> "$OUT/nproc.txt"

if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke rc=$?" >> "$OUT/smoke.log"
fi

timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench rc=$?" >> "$OUT/bench.err"
if [ -z "${SKIP_REF:-}" ]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
fi

# launch list (cold-cache, serialised): shares per kernel, not absolutes
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exchange \
  > "$OUT/launches_bench.log" 2>&1
python tests/launch_breakdown.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1

# one full capture of the SpMM: one epoch worth of launches after warm-up
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 24 -c 8 \
  -o "$OUT/prof_spmm" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-exchange \
  > "$OUT/prof_spmm.log" 2>&1
if [ -z "${SKIP_GEMM_PROF:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 18 -c 3 \
    -o "$OUT/prof_gemm" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-exchange \
    > "$OUT/prof_gemm.log" 2>&1
fi
echo done > "$OUT/DONE"
