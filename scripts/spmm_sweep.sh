# SpMM configuration sweep on C2 (bench's per-launch CUDA-event times), one
# bench process per setting.  CONFIGS: space-separated "VAR=val,VAR=val" items
O=gpurun_out/${SWEEP_OUT:-sweep}
mkdir -p $O
for c in ${CONFIGS:-CG_SPMM_FLAGS=0 CG_SPMM_FLAGS=1}; do
  envs=$(echo $c | tr ',' ' ')
  tag=$(echo $c | tr ',=' '__')
  env $envs timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exchange \
    > $O/$tag.json 2> $O/$tag.err
  python - "$O/$tag.json" "$c" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[2], "epoch_ms %.4f" % d["ms_per_step"],
          "spmm_ms %.4f" % r["spmm_ms_per_epoch"], [l["ms"] for l in r["launches"]], flush=True)
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done | tee $O/summary.txt
