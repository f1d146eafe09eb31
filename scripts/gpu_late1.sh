#!/bin/bash
# Late phases: parity first, then A/B on the configs (kernel ms, phases).
O=gpurun_out/late1; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader > $O/gpu.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "late_phase" > $O/pytest.log 2>&1
tail -5 $O/pytest.log
for c in C5 C2; do
  timeout 900 python scripts/tune.py $c --reps 8 BM_LATE=0 BM_LATE=1 BM_LATE=1,BM_LATE_ROOTS=8192 > $O/tune_$c.json 2>&1
  tail -3 $O/tune_$c.json | cut -c1-400
done
timeout 600 python scripts/tune.py C5 --reps 2 --tl BM_LATE=1 > $O/tl_C5.json 2>&1
tail -c 3000 $O/tl_C5.json
