O=gpurun_out/r3l
mkdir -p $O
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $O/c4_nch1_5blk.json 2> $O/c4.err
python tests/bench_spmm.py 2449029 26.25 100 > $O/spmm100.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k spmm > $O/pytest.log 2>&1
