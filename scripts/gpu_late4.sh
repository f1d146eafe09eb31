#!/bin/bash
O=gpurun_out/late4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "late_phase" > $O/pytest.log 2>&1
tail -3 $O/pytest.log
timeout 600 python scripts/late_tl.py C5 --reps 3 > $O/C5.txt 2>&1; cut -c1-900 $O/C5.txt
timeout 300 python scripts/late_tl.py C2 --reps 3 > $O/C2.txt 2>&1; cut -c1-600 $O/C2.txt
for c in C5 C2; do
  timeout 900 python scripts/tune.py $c --reps 10 BM_LATE=0 BM_LATE=1 > $O/tune_$c.json 2>&1
  python - $O/tune_$c.json <<'PY'
import json, sys, statistics
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line); print(d["cfg"], d["spec"], "mean %.2f" % statistics.mean(d["ms"]), "min", d["ms_min"], d["phases"], d["ok"])
PY
done
