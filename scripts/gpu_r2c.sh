set -x
O=gpurun_out/r2c
mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_golden_big.py tests/test_gpu_train_parity.py -q --durations=20 > $O/pytest_new.log 2>&1
echo "pytest rc $?" >> $O/pytest_new.log
for b in 16 32 64; do
  CG_WT_BLOCKS=$b timeout 300 python scripts/exchange_probe.py 14 > $O/wt_blocks_$b.log 2>&1
done
SWEEP_OUT=r2c/sweep bash scripts/spmm_sweep.sh > $O/sweep.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_gemm_tc --launch-skip 40 -c 8 -o $O/ncu_gemm python bench.py --steps 2 --warmup 5 --no-cpu-baseline --no-exchange > $O/ncu_gemm.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
