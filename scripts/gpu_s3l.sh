# session 3: lazy roots — GPU suite, C5 A/B against a no-lazy build, host copy rates
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python scripts/host_copy_rate.py > gpurun_out/s3l_copyrate.txt 2>&1; cat gpurun_out/s3l_copyrate.txt
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/s3l_pytest.log 2>&1; tail -2 gpurun_out/s3l_pytest.log
REPS=8 bash scripts/gpu_ab.sh s3l C5 nolazy > /dev/null 2>&1
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob('gpurun_out/s3l_C*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    pp = [m / p for m, p in zip(d['ms'], d['phases'])]
    print(f, d['ms_med'], d['phases'], 'ms/phase %.2f' % statistics.median(pp), d['ok'],
          {k: round(v / 1000, 1) for k, v in d['timeline']['per_kind_us'].items() if v > 500})
PY
