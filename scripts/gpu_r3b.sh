O=gpurun_out/r3b
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k spmm > $O/pytest.log 2>&1
for v in "" "CG_SPMM_G2=1" "" "CG_SPMM_G2=1"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-exchange --steps 20 >> "$O/b_${v:-default}.jsonl" 2>> $O/err.log
done
CG_SPMM_G2=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k spmm > $O/pytest_g2.log 2>&1
