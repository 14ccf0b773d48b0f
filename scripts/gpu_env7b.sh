#!/bin/bash
# Llama-7B shape (B=12): stream-overlap switches A/B under accumulation (one B200).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e7
run() {
  env $1 timeout 900 python bench.py --config llama-7b --grad-accum 4 --steps 3 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/e7/$2.json > /dev/null 2>&1
  python - "$2" "$1" <<'PY'
import json, sys
l = json.load(open(f"gpurun_out/e7/{sys.argv[1]}.json"))["line"]
print(sys.argv[2], round(l["value"]), round(l["mfu"] * 100, 2), l["clocks"]["sm_mhz"])
PY
}
for rep in 1 2; do
  run "QTB_NONE=0" base_$rep
  run "QTB_ATTN_2S=0" a2s_$rep
  run "QTB_WGRAD_SIDE=0" side_$rep
done
