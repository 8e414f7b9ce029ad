set -x
O=gpurun_out/r2d
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q --durations=25 > $O/pytest_gpu.log 2>&1
echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm --launch-skip 24 -c 8 -o $O/ncu_spmm python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exchange > $O/ncu_spmm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc --launch-skip 24 -c 8 -o $O/ncu_gemm python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exchange > $O/ncu_gemm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
