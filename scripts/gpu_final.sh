#!/usr/bin/env bash
# One gpurun call: the round's evidence -- GPU parity suite, smoke, the bench
# line (both arms), C3 / C4 lines, a 2-rank (one GPU, gloo) exchange line, the
# launch list and ncu captures of the SpMM and the GEMM.
#   gpurun --timeout 5400 -- 'bash scripts/gpu_final.sh r02_final'
set -u
TAG=${1:-r02_final}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"; grep -m1 "model name" /proc/cpuinfo >> "$OUT/nproc.txt"; free -g >> "$OUT/nproc.txt"
timeout 2400 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
timeout 900 python bench.py --config c4 --no-cpu-baseline > "$OUT/bench_c4.json" 2> "$OUT/bench_c4.err"
timeout 900 python bench.py --config c3 --no-cpu-baseline > "$OUT/bench_c3.json" 2> "$OUT/bench_c3.err"
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 5 --no-cpu-baseline > "$OUT/bench_2rank_gloo.json" 2> "$OUT/bench_2rank.err"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exchange \
  > "$OUT/launches_bench.log" 2>&1
python tests/launch_breakdown.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 24 -c 8 \
  -o "$OUT/prof_spmm" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-exchange \
  > "$OUT/prof_spmm.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 24 -c 8 \
  -o "$OUT/prof_gemm" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-exchange \
  > "$OUT/prof_gemm.log" 2>&1
echo done > "$OUT/DONE"
