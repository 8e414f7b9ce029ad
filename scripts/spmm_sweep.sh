# SpMM store/gather cache-policy and column-slice sweep on C2 (bench's
# per-launch CUDA-event times), one bench process per setting
O=gpurun_out/${SWEEP_OUT:-sweep}
mkdir -p $O
for slice in ${SLICES:-128 64}; do
  for flags in ${FLAGS:-0 1 2 4 5}; do
    CG_SPMM_SLICE=$slice CG_SPMM_FLAGS=$flags timeout 300 python bench.py --steps 10 --warmup 3 \
      --no-cpu-baseline --no-exchange > $O/s${slice}_f${flags}.json 2> $O/s${slice}_f${flags}.err
    python - "$O/s${slice}_f${flags}.json" "$slice" "$flags" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print("slice", sys.argv[2], "flags", sys.argv[3], "epoch_ms %.4f" % d["ms_per_step"],
          "spmm_ms %.4f" % r["spmm_ms_per_epoch"], [l["ms"] for l in r["launches"]], flush=True)
except Exception as e:
    print("slice", sys.argv[2], "flags", sys.argv[3], "failed", e)
PY
  done
done | tee $O/summary.txt
