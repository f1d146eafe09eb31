# session 3: bucketed pushed levels in the push-only kernels (C4, C3, C1 push; interleaved row state only on C4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bucketed or corpus_given or planted" 2>&1 | tail -1
for c in C4 C3 C1; do
  timeout 600 python scripts/tune.py $c --reps 10 - BM_PB=0 > gpurun_out/s3z_$c.json 2>&1
  BM_LIB=tunelib/prev.so timeout 600 python scripts/tune.py $c --reps 10 - > gpurun_out/s3z_${c}_prev.json 2>&1
done
python - <<'PY'
import json, statistics, glob
for f in sorted(glob.glob('gpurun_out/s3z_C*.json')):
    for l in open(f):
        if not l.startswith('{'): continue
        d = json.loads(l); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
        print(f.split('/')[-1], d['spec'], 'mean %.2f' % statistics.mean(d['ms']), d['phases'], 'ms/phase %.3f' % statistics.median(pp), d['ok'])
PY
