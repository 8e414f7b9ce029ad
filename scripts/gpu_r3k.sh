O=gpurun_out/r3k
mkdir -p $O
timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/c3_4blk.json 2> $O/c3.err
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k spmm > $O/pytest.log 2>&1
