# session 3: leftover lists — parity, A/B against BM_BU_LEFT=0 (C5, C2); C5 launch list covering the timed steps
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_upload.py -x -q -k "bottom_up or lazy or mixed or bucketed or prebuilt" > gpurun_out/s3t_pytest.log 2>&1; tail -1 gpurun_out/s3t_pytest.log
timeout 1500 python scripts/tune.py C5 --tl --reps 8 - BM_BU_LEFT=0 > gpurun_out/s3t_c5.json 2>&1
timeout 600 python scripts/tune.py C2 --tl --reps 8 - BM_BU_LEFT=0 > gpurun_out/s3t_c2.json 2>&1
python - <<'PY'
import json, statistics
for f in ('gpurun_out/s3t_c5.json', 'gpurun_out/s3t_c2.json'):
    for l in open(f):
        if not l.startswith('{'): continue
        d = json.loads(l); pp = [m / p for m, p in zip(d['ms'], d['phases'])]
        print(d['cfg'], d['spec'], 'med', d['ms_med'], d['phases'], 'ms/phase %.2f' % statistics.median(pp), d['ok'],
              {k: round(v / 1000, 1) for k, v in d['timeline']['per_kind_us'].items() if v > 300})
PY
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/s3t_c5_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-alt --no-e2e > gpurun_out/s3t_launches_bench.log 2>&1; echo "ncu rc=$?"
