O=gpurun_out/r2p
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench$i.json 2> $O/bench$i.err
CG_SPMM_LANES=16 timeout 900 python bench.py --no-cpu-baseline --no-exchange > $O/bench_l16_$i.json 2> $O/bench_l16_$i.err
done
