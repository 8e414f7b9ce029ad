O=gpurun_out/r3c
mkdir -p $O
timeout 600 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c1 --impl reference --steps 2 > $O/bench_c1_ref.json 2> $O/bench_c1_ref.err
timeout 600 python tests/diag_c1_tfl.py > $O/diag_c1_tfl.txt 2>&1
