# round 2: new parity tests (C2 float on both cache configs, C3/C4 goldens,
# write-through queue), bench with the exchange queue, sanitizers, K3 ncu
set -x
O=gpurun_out/r2b
mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_train_parity.py tests/test_gpu_golden_big.py -x -q --durations=15 > $O/pytest_new.log 2>&1
echo "pytest rc $?" >> $O/pytest_new.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_${tool}_smoke.log 2>&1
  echo "rc $?" >> $O/sanitizer_${tool}_smoke.log
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -x -q > $O/sanitizer_memcheck_kernels.log 2>&1
echo "rc $?" >> $O/sanitizer_memcheck_kernels.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm_tcgen05 or wgrad_tcgen05 or softmax or spmm" > $O/sanitizer_racecheck_kernels.log 2>&1
echo "rc $?" >> $O/sanitizer_racecheck_kernels.log
timeout 900 ncu --set full --import-source on -k regex:k_copy_rows --launch-skip 40 -c 6 -o $O/ncu_k3 python scripts/exchange_probe.py 12 > $O/ncu_k3.log 2>&1
