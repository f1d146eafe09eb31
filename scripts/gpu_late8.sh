#!/bin/bash
O=gpurun_out/late8; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "late_phase" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in base lt1 lt4; do
  if [ $v = base ]; then L=""; else L="tunelib/$v.so"; fi
  BM_LIB=$L timeout 600 python scripts/tune.py C5 --reps 10 - > $O/tune_C5_$v.json 2>&1
  BM_LIB=$L timeout 600 python scripts/tune.py C2 --reps 10 - > $O/tune_C2_$v.json 2>&1
done
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob("gpurun_out/late8/tune_*.json")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); print(f.split("/")[-1], "mean %.2f" % statistics.mean(d["ms"]), "min", d["ms_min"], d["phases"], d["ok"])
PY
BM_LIB=tunelib/lt1.so timeout 300 python scripts/late_tl.py C5 --reps 1 > $O/C5_lt1.txt 2>&1; cut -c1-700 $O/C5_lt1.txt
timeout 300 python scripts/late_tl.py C5 --reps 1 > $O/C5.txt 2>&1; cut -c1-700 $O/C5.txt
