O=gpurun_out/r3e
mkdir -p $O
for v in "" "CG_WGRAD_TILES_PER_SM=1" "" "CG_WGRAD_TILES_PER_SM=1" "" "CG_WGRAD_TILES_PER_SM=1"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-exchange --steps 20 >> "$O/b_${v:-default}.jsonl" 2>> $O/err.log
done
