O=gpurun_out/r2r
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
cat /sys/bus/pci/devices/*/numa_node > $O/numa_nodes.txt 2>&1
python tests/diag_e2e.py > $O/diag_e2e.txt 2>&1
for n in 0 1; do numactl --cpunodebind=$n --membind=$n python tests/diag_e2e.py > $O/diag_e2e_node$n.txt 2>&1; done
python -m pytest tests/test_gpu_kernels.py -q -k "wgrad or tcgen05" > $O/pytest_gemm.log 2>&1
python tests/bench_gemm.py wgrad2:1 fwd2:1pre > $O/gemm_narrow.txt 2>&1
