O=gpurun_out/r2q
mkdir -p $O
for v in "" "CG_SPMM_SLICE=96" "CG_SPMM_SLICE=88" "CG_SPMM_SLICE=64" "CG_SPMM_FLAGS=5" "CG_SPMM_FLAGS=0" "CG_SPMM_S=6" ""; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-exchange --steps 20 > "$O/b_${v:-default}.json" 2>> $O/err.log
done
