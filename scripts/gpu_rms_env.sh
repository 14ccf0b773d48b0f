#!/bin/bash
# RMSNorm path / staging A/B on the 0.5B bench (GA=1), env switches only.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rms
run() {
  env $1 timeout 600 python bench.py --grad-accum 1 --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/rms/$2.json > /dev/null 2>&1
  python - "$2" "$1" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/rms/{sys.argv[1]}.json"))
l = d["line"]; k = l["kernel_classes"]
print(sys.argv[2], round(l["value"]), round(l["ms_per_step"], 2), l["clocks"]["sm_mhz"], "rmsnorm", k["rmsnorm"]["ms"], "quant", k["quant"]["ms"])
PY
}
for rep in 1 2; do
  run "QTB_RF_SMEM=100" base_$rep
  run "QTB_RF_SMEM=58" r16_$rep
  run "QTB_RF_MIN_ROWS=100000" stream_$rep
done
