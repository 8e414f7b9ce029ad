O=gpurun_out/r2s
mkdir -p $O
for i in 1 2 3 4; do
  timeout 600 python bench.py --no-cpu-baseline --no-exchange > $O/b$i.json 2>> $O/err.log
done
timeout 900 python bench.py > $O/full.json 2>> $O/err.log
