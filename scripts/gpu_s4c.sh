# session 3: more out-of-line choices in the pulled-capable kernels (C5, C2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in C5 C2; do
  for v in base pbinline sweepni; do
    if [ $v = base ]; then L=""; else L="tunelib/$v.so"; fi
    BM_LIB=$L timeout 900 python scripts/tune.py $c --reps 12 - > gpurun_out/s4c_${c}_$v.json 2>&1
  done
done
python - <<'PY'
import json, statistics, glob
for f in sorted(glob.glob('gpurun_out/s4c_C*.json')):
    d = json.loads(open(f).read().strip().splitlines()[-1]); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
    print(f.split('/')[-1], 'mean %.2f' % statistics.mean(d['ms']), d['phases'], 'ms/phase %.3f' % statistics.median(pp), d['ok'])
PY
