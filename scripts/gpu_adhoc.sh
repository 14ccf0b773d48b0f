#!/bin/bash
QTB_ATTN_NOWAIT=0 timeout 300 python scripts/attn_nowait.py
QTB_ATTN_NOWAIT=1 timeout 300 python scripts/attn_nowait.py
python - <<'PY'
import torch, glob
for f in sorted(glob.glob("/tmp/fwd_0_*.pt")):
    a = torch.load(f); b = torch.load(f.replace("fwd_0_", "fwd_1_"))
    print(f, "nowait vs wait bitwise:", all(torch.equal(x, y) for x, y in zip(a, b)))
PY
