O=gpurun_out/r2v
mkdir -p $O
for v in "" "CG_SPMM_FLAGS=24577" "CG_SPMM_FLAGS=16385" "CG_SPMM_FLAGS=8193" "CG_SPMM_FLAGS=5" ""; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-exchange --steps 20 > "$O/b_${v:-default}.json" 2>> $O/err.log
done
