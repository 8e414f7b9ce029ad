# C3 regression hunt: round-1 code (worktree r01tree) vs HEAD with the
# transform-first paths off, same box
O=gpurun_out/r3g
mkdir -p $O
(cd r01tree && timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > ../$O/c3_r01.json 2> ../$O/c3_r01.err)
CG_SAGE_TF0=0 CG_TFL=0 timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 10 > $O/c3_head_agg.json 2> $O/c3_head_agg.err
