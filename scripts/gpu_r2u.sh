# compute-sanitizer over the kernel tests (every kernel, including this
# round's epilogue variants, resident-B GEMMs, mask bits, ReLU bits) and smoke
O=gpurun_out/r2u
mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -x -q > $O/sanitizer_memcheck_kernels.log 2>&1
echo "rc $?" >> $O/sanitizer_memcheck_kernels.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or wgrad or softmax or spmm or relu" > $O/sanitizer_racecheck_kernels.log 2>&1
echo "rc $?" >> $O/sanitizer_racecheck_kernels.log
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or wgrad or spmm" > $O/sanitizer_synccheck_kernels.log 2>&1
echo "rc $?" >> $O/sanitizer_synccheck_kernels.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_${tool}_smoke.log 2>&1
  echo "rc $?" >> $O/sanitizer_${tool}_smoke.log
done
# the SAGE layer-0 transform-first and GCN last-layer transform-first epochs
CG_GCN_TFL=1 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_train_parity.py -x -q -k "transform_first" > $O/sanitizer_memcheck_transform_first.log 2>&1
echo "rc $?" >> $O/sanitizer_memcheck_transform_first.log
