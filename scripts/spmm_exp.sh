set -u
OUT=gpurun_out/${1:-sx}; mkdir -p $OUT
CG_SPMM_TMA=1 CG_SPMM_TMA_W=8 CG_SPMM_TMA_D=4 timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k "spmm" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
grep -q "rc=0" $OUT/pytest_k.log || exit 0
CG_SPMM_TMA=0 timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_lsu.json 2>> $OUT/bench.err
for wd in 4,8 8,4 16,2 8,8 16,4 4,16; do W=${wd%,*}; D=${wd#*,}
CG_SPMM_TMA=1 CG_SPMM_TMA_W=$W CG_SPMM_TMA_D=$D timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_${W}_${D}.json 2>> $OUT/bench.err; done
