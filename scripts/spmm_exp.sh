set -u
OUT=gpurun_out/${1:-sx}; mkdir -p $OUT
for ss in 8,6 8,4 8,3 16,4 4,4 12,4 8,8; do S1=${ss%,*}; S2=${ss#*,}
CG_SPMM_ASYNC=1 CG_SPMM_S1=$S1 CG_SPMM_S2=$S2 timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_${S1}_${S2}.json 2>> $OUT/bench.err; done
