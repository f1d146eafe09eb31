#!/bin/bash
O=gpurun_out/late12; mkdir -p $O
timeout 900 python scripts/tune.py C5 --reps 12 - BM_LATE_BCAP=1000000 BM_LATE_BCAP=1500000 BM_LATE_BCAP=1500000,BM_LATE_FPER=2048 > $O/tune_C5.json 2>&1
timeout 900 python scripts/tune.py C2 --reps 16 - BM_LATE_BCAP=500000 BM_LATE_BCAP=1000000 BM_LATE_BCAP=1500000 > $O/tune_C2.json 2>&1
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob("gpurun_out/late12/tune_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "med", d["ms_med"], d["phases"], d["ok"])
PY
timeout 300 python scripts/late_tl.py C2 --reps 2 > $O/C2_def.txt 2>&1; cut -c1-700 $O/C2_def.txt
timeout 300 python scripts/late_tl.py C2 --reps 2 BM_LATE_BCAP=1000000 > $O/C2_b1m.txt 2>&1; cut -c1-700 $O/C2_b1m.txt
