O=gpurun_out/r3h
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q > $O/pytest_kernels.log 2>&1
echo "rc $?" >> $O/pytest_kernels.log
timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/c3.json 2> $O/c3.err
CG_SAGE_TF0=0 CG_TFL=0 timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/c3_agg.json 2> $O/c3_agg.err
timeout 600 python bench.py --no-cpu-baseline --no-exchange > $O/c2.json 2> $O/c2.err
