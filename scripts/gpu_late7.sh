#!/bin/bash
O=gpurun_out/late7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "late_phase" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for c in C5 C2; do
timeout 900 python scripts/tune.py $c --reps 10 - BM_LATE=0 > $O/tune_$c.json 2>&1
python - $O/tune_$c.json <<'PY'
import json, sys, statistics
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "min", d["ms_min"], d["phases"], d["ok"])
PY
done
