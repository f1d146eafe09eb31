# session 3: two candidates per lane in pulled sweeps (slots2, slots2 at 2 CTAs/SM) — parity then C5/C2 A/B
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
BM_LIB=tunelib/slots2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bottom_up or lazy or mixed or bucketed" > gpurun_out/s3j_pytest.log 2>&1; tail -1 gpurun_out/s3j_pytest.log
REPS=6 bash scripts/gpu_ab.sh s3j C5 slots2 slots2m2 > /dev/null 2>&1
REPS=6 bash scripts/gpu_ab.sh s3j C2 slots2 > /dev/null 2>&1
python - <<'PY'
import json, glob, statistics
for f in sorted(glob.glob('gpurun_out/s3j_C*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    pp = [m / p for m, p in zip(d['ms'], d['phases'])]
    print(f, d['ms_med'], d['phases'], 'ms/phase %.2f' % statistics.median(pp), d['ok'],
          {k: round(v / 1000, 1) for k, v in d['timeline']['per_kind_us'].items() if v > 500})
PY
