set -u
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "wgrad" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
for r in 1 2; do
(cd ab_head && timeout 200 python tests/bench_gemm.py wgrad2:1 wgrad1:1 wgrad0:1 > ../$OUT/gemm_head_$r.txt 2>&1)
timeout 200 python tests/bench_gemm.py wgrad2:1 wgrad1:1 wgrad0:1 > $OUT/gemm_new_$r.txt 2>&1
(cd ab_head && timeout 300 python bench.py --no-cpu-baseline --steps 20 > ../$OUT/bench_head_$r.json 2>/dev/null)
timeout 300 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_new_$r.json 2>/dev/null
done
