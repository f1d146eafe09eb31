#!/bin/bash
# push-only configs: pulled-capable kernel (row index) with and without late phases against the default push kernel
O=gpurun_out/late5; mkdir -p $O
for c in C3 C4 C1; do
  timeout 900 python scripts/tune.py $c --reps 10 - TUNE_BU=on,BM_LATE=0 TUNE_BU=on,BM_LATE=1 TUNE_BU=on,BM_LATE=1,BM_BU_FRAC=2 > $O/tune_$c.json 2>&1
  python - $O/tune_$c.json <<'PY'
import json, sys, statistics
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "min", d["ms_min"], d["phases"], d["ok"])
    elif "Error" in line or "error" in line: print(line[:300])
PY
done
timeout 300 python scripts/late_tl.py C3 --reps 2 > $O/C3.txt 2>&1; cut -c1-700 $O/C3.txt
