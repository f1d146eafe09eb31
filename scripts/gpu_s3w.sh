# session 3: WR filtering at hit/claim time — phase counts and per-phase cost on C5 (10 runs each)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python scripts/tune.py C5 --tl --reps 10 - BM_CLAIM_MODE=1 > gpurun_out/s3w_base.json 2>&1
BM_LIB=tunelib/deadhit.so timeout 1200 python scripts/tune.py C5 --tl --reps 10 - BM_CLAIM_MODE=1 > gpurun_out/s3w_deadhit.json 2>&1
python - <<'PY'
import json, statistics
for f in ('gpurun_out/s3w_base.json', 'gpurun_out/s3w_deadhit.json'):
    for l in open(f):
        if not l.startswith('{'): continue
        d = json.loads(l); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
        lv = d['timeline']['levels']; roots = []; last = -1
        for x in lv:
            if x[0] != last: roots.append(x[1]); last = x[0]
        print(f.split('/')[-1], d['spec'], 'mean %.2f' % statistics.mean(d['ms']), 'med', d['ms_med'], 'phases mean %.2f' % statistics.mean(d['phases']), d['phases'], 'ms/phase %.2f' % statistics.median(pp), d['ok'], roots)
PY
