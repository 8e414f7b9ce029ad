set -u
OUT=gpurun_out/${1:-sx}; mkdir -p $OUT
for v in 1 2 3 4; do
  CG_WGRAD_TILES_PER_SM=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$v.json 2>> $OUT/bench.err
  CG_WGRAD_TILES_PER_SM=$v timeout 120 python tests/bench_gemm.py wgrad1:1 wgrad0:1 wgrad2:1 > $OUT/gemm_$v.txt 2>&1
done
