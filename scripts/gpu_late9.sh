#!/bin/bash
O=gpurun_out/late9; mkdir -p $O
timeout 900 python scripts/tune.py C5 --reps 8 - BM_LATE_ROOTS=5000000,BM_LATE_BCAP=5000000 BM_LATE_ROOTS=5000000,BM_LATE_BCAP=5000000,BM_LATE_FCAP=64000000 > $O/tune_C5.json 2>&1
timeout 900 python scripts/tune.py C2 --reps 8 - BM_LATE_ROOTS=5000000,BM_LATE_BCAP=5000000 > $O/tune_C2.json 2>&1
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob("gpurun_out/late9/tune_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "min", d["ms_min"], d["phases"], d["ok"])
PY
timeout 300 python scripts/late_tl.py C5 --reps 1 BM_LATE_ROOTS=5000000 BM_LATE_BCAP=5000000 > $O/C5_r5m.txt 2>&1; cut -c1-900 $O/C5_r5m.txt
