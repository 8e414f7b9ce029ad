O=gpurun_out/r3a
mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c4.log 2>&1
python tests/launch_breakdown.py $O/launches_c4.csv > $O/launches_c4_summary.txt 2>&1
