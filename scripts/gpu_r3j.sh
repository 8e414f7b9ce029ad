O=gpurun_out/r3j
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
timeout 900 python bench.py --config c4 --no-cpu-baseline --steps 10 > $O/c4.json 2> $O/c4.err
timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/c3.json 2> $O/c3.err
timeout 600 python bench.py --no-cpu-baseline --no-exchange > $O/c2.json 2> $O/c2.err
