#!/bin/bash
O=gpurun_out/late11; mkdir -p $O
timeout 900 python scripts/tune.py C5 --reps 10 - BM_BU_ALPHA=6 BM_BU_ALPHA=10 BM_BU_ALPHA=12 BM_LATE_BCAP=3000000 BM_LATE_BCAP=1500000 BM_LATE_FPER=2048 > $O/tune_C5.json 2>&1
timeout 900 python scripts/tune.py C2 --reps 10 - BM_BU_ALPHA=3 BM_BU_ALPHA=6 BM_LATE_BCAP=1000000 BM_LATE_BCAP=4000000 > $O/tune_C2.json 2>&1
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob("gpurun_out/late11/tune_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "med", d["ms_med"], d["phases"], d["ok"])
PY
