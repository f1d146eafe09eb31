# session 3: expand_level out of line in the pulled-capable kernels — parity, then against the previous build
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for c in C5 C2 C4 C3; do
  timeout 900 python scripts/tune.py $c --reps 12 - > gpurun_out/s4b_${c}_new.json 2>&1
  BM_LIB=tunelib/prev.so timeout 900 python scripts/tune.py $c --reps 12 - > gpurun_out/s4b_${c}_prev.json 2>&1
done
python - <<'PY'
import json, statistics, glob
for f in sorted(glob.glob('gpurun_out/s4b_C*.json')):
    d = json.loads(open(f).read().strip().splitlines()[-1]); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
    print(f.split('/')[-1], 'mean %.2f' % statistics.mean(d['ms']), d['phases'], 'ms/phase %.3f' % statistics.median(pp), d['ok'])
PY
