set -x
O=gpurun_out/r2e
mkdir -p $O
SWEEP_OUT=r2e/sweep CONFIGS="CG_SPMM_SLICE=128 CG_SPMM_SLICE=128,CG_SPMM_LANES=8 CG_SPMM_SLICE=128,CG_SPMM_LANES=4 CG_SPMM_SLICE=64 CG_SPMM_SLICE=64,CG_SPMM_LANES=4 CG_SPMM_SLICE=0 CG_SPMM_SLICE=0,CG_SPMM_LANES=16 CG_SPMM_SLICE=0,CG_SPMM_LANES=8 CG_SPMM_SLICE=128,CG_SPMM_LANES=8,CG_SPMM_S=6 CG_SPMM_SLICE=64,CG_SPMM_LANES=4,CG_SPMM_S=6" bash scripts/spmm_sweep.sh > $O/sweep.log 2>&1
CG_SPMM_SLICE=64 CG_SPMM_LANES=4 timeout 600 ncu --set full --clock-control none -k regex:k_spmm --launch-skip 24 -c 8 -o $O/ncu_spmm_s64l4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exchange > $O/ncu1.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_golden_big.py tests/test_gpu_train_parity.py tests/test_gpu_graphs.py -q -x > $O/pytest.log 2>&1
echo "rc $?" >> $O/pytest.log
