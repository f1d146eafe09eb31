# session 3: pull-rule alpha sweep now that wide pushed levels are bucketed (C5); C2 alpha too
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python scripts/tune.py C5 --reps 8 BM_BU_ALPHA=6 BM_BU_ALPHA=8 BM_BU_ALPHA=10 BM_BU_ALPHA=12 - > gpurun_out/s3n_alpha_c5.json 2>&1
timeout 600 python scripts/tune.py C2 --reps 8 BM_BU_ALPHA=2 BM_BU_ALPHA=3 - BM_BU_ALPHA=6 > gpurun_out/s3n_alpha_c2.json 2>&1
python - <<'PY'
import json, statistics
for f in ('gpurun_out/s3n_alpha_c5.json', 'gpurun_out/s3n_alpha_c2.json'):
    for l in open(f):
        if not l.startswith('{'): continue
        d = json.loads(l); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
        print(d['cfg'], d['spec'], 'med', d['ms_med'], 'mean %.2f' % statistics.mean(d['ms']), d['phases'], 'ms/phase %.2f' % statistics.median(pp), d['ok'])
PY
