O=gpurun_out/r3d
mkdir -p $O
for t in 1 2 3 4; do CG_WGRAD_TILES_PER_SM=$t python tests/bench_gemm.py wgrad2:1 wgrad1:1 wgrad0:1 > $O/wgrad_t$t.txt 2>&1; done
for st in 3 4; do CG_GEMM_STAGES=$st python tests/bench_gemm.py wgrad2:1 wgrad1:1 wgrad0:1 fwd1:1pre > $O/stages_$st.txt 2>&1; done
