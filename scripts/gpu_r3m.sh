O=gpurun_out/r3m
mkdir -p $O
for v in "" "CG_SPMM_S=3" "" "CG_SPMM_S=3"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-exchange --steps 20 >> "$O/b_${v:-default}.jsonl" 2>> $O/err.log
done
