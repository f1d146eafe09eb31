#!/bin/bash
O=gpurun_out/late13; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "late_phase" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 900 python scripts/tune.py C5 --reps 12 - > $O/tune_C5.json 2>&1
timeout 900 python scripts/tune.py C2 --reps 16 - > $O/tune_C2.json 2>&1
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob("gpurun_out/late13/tune_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "med", d["ms_med"], d["phases"], d["ok"])
PY
