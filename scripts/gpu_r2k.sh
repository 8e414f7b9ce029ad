O=gpurun_out/r2k
mkdir -p $O
for cfg in "" "CG_SPMM_ASYNC=1" "CG_SPMM_ASYNC=1 CG_SPMM_LANES=4" "CG_SPMM_ASYNC=1 CG_SPMM_LANES=16" "CG_SPMM_ASYNC=1 CG_SPMM_S=8" "CG_SPMM_ASYNC=1 CG_SPMM_G4=0" "CG_SPMM_FLAGS=0" "CG_SPMM_ASYNC=1 CG_SPMM_FLAGS=0"; do
  env $cfg python tests/bench_spmm.py 2449029 26.25 48 100 256 >> $O/spmm_c4.txt 2>&1
done
timeout 900 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
