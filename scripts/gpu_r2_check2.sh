cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
./scripts/ubench_corun > gpurun_out/c2_corun.txt 2>&1; cat gpurun_out/c2_corun.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c2_smoke.log 2>&1; tail -1 gpurun_out/c2_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c2_pytest.log 2>&1; tail -2 gpurun_out/c2_pytest.log
for c in C1 C2 C3 C4 C5; do timeout 600 python scripts/tune.py $c --reps 6 - 2>&1 | tail -1 | python -c "import json,sys,statistics; d=json.loads(sys.stdin.read()); pp=[m/p for m,p in zip(d['ms'],d['phases'])]; print(d['cfg'], d['ms_med'], d['phases'], 'ms/phase %.3f'%statistics.median(pp), d['ok'])"; done
