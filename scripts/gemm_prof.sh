set -u
OUT=gpurun_out/${1:-gp}; mkdir -p $OUT
python tests/bench_gemm.py > $OUT/bench_gemm.txt 2>&1
for c in ${CASES:-fwd1:1pre fwd1:2 dgrad2:1pre wgrad1:1}; do
  n=${c/:/_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 2 -c 1 \
    -o $OUT/prof_$n python tests/bench_gemm.py $c > $OUT/prof_$n.log 2>&1
done
