# session 3: bucketed pushed levels — parity, then A/B against BM_PB=0 on C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bucketed or bottom_up or lazy or mixed" > gpurun_out/s3i_pytest.log 2>&1; tail -3 gpurun_out/s3i_pytest.log
timeout 1200 python scripts/tune.py C5 --tl --reps 6 - BM_PB=0 BM_PB_MIN=16000000 > gpurun_out/s3i_ab.json 2>&1
python - <<'PY'
import json, statistics
for l in open('gpurun_out/s3i_ab.json'):
    if not l.startswith('{'): print(l.strip()[:300]); continue
    d = json.loads(l); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
    tl = d.get('timeline', {})
    print(d['spec'], d['ms_med'], d['phases'], 'ms/phase %.2f' % statistics.median(pp), d['ok'],
          {k: round(v / 1000, 1) for k, v in tl.get('per_kind_us', {}).items() if v > 200})
    for lv in tl.get('levels', []):
        if lv[2] > 1500: print('   ', lv)
PY
