#!/bin/bash
O=gpurun_out/late6; mkdir -p $O
timeout 900 python scripts/tune.py C5 --reps 10 - BM_LATE_BCAP=600000 BM_LATE_BCAP=8000000 BM_LATE_ROOTS=500000,BM_LATE_FCAP=16000000 BM_LATE_ROOTS=500000,BM_LATE_FCAP=16000000,BM_LATE_BCAP=8000000 BM_LATE_FPER=256 BM_LATE_FPER=4096 > $O/tune_C5.json 2>&1
python - $O/tune_C5.json <<'PY'
import json, sys, statistics
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "min", d["ms_min"], d["phases"], d["ok"])
PY
timeout 300 python scripts/late_tl.py C5 --reps 2 BM_LATE_ROOTS=500000 BM_LATE_FCAP=16000000 > $O/C5_r500k.txt 2>&1; cut -c1-900 $O/C5_r500k.txt
