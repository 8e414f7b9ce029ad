# e2e variance probe: the bench's e2e record (host enqueue, bare input H2D)
# three times on whatever box this call lands on
O=gpurun_out/e2e_probe_$1
mkdir -p $O
nvidia-smi -q | grep -iE "Bus Id|Link Width|Link Gen|Max Link" > $O/pcie.txt 2>&1
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-exchange --steps 20 >> $O/bench.jsonl 2>> $O/err.log; done
