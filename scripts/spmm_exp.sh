set -u
OUT=gpurun_out/${1:-sx}; mkdir -p $OUT
CG_SPMM_SLICE=64 timeout 300 python -m pytest tests/test_gpu_train_parity.py -x -q -k "c2" > $OUT/pytest_t.log 2>&1; echo "rc=$?" >> $OUT/pytest_t.log
for cfg in "0 -1" "128 -1" "64 -1" "64 1"; do set -- $cfg
if [ "$2" = "-1" ]; then CG_SPMM_SLICE=$1 timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$1_$2.json 2>> $OUT/bench.err
else CG_SPMM_SLICE=$1 CG_SPMM_ASYNC=$2 timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$1_$2.json 2>> $OUT/bench.err; fi; done
