#!/usr/bin/env bash
# Same-box A/B of the working tree against a committed baseline.
#   git worktree add -f ab_head <rev> && (cd ab_head && python -m paper_2508_13716_b200.build)
#   gpurun -- 'bash scripts/ab.sh TAG [reps] [bench args...]'
# Runs bench.py (and the GEMM microbenchmark) alternately in ab_head/ (A) and
# the working tree (B) on the same GPU, so box-to-box variation cancels.
set -u
TAG=${1:-ab}; REPS=${2:-2}; shift 2 || true
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in $(seq 1 $REPS); do
  (cd ab_head && timeout 300 python bench.py --no-cpu-baseline --steps 20 "$@" > ../$OUT/bench_A_$r.json 2>/dev/null)
  timeout 300 python bench.py --no-cpu-baseline --steps 20 "$@" > $OUT/bench_B_$r.json 2>/dev/null
  (cd ab_head && timeout 200 python tests/bench_gemm.py fwd0:1pre fwd1:1pre dgrad2:1pre wgrad1:1 > ../$OUT/gemm_A_$r.txt 2>&1)
  timeout 200 python tests/bench_gemm.py fwd0:1pre fwd1:1pre dgrad2:1pre wgrad1:1 > $OUT/gemm_B_$r.txt 2>&1
done
