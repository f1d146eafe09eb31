# session 3: prefetch A/B on C5 + cycle split; bench contract (new e2e legs); racecheck with a 1-CTA grid
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
BM_LIB=tunelib/pf.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bottom_up or lazy or mixed" > gpurun_out/s3g_pytest_pf.log 2>&1; tail -1 gpurun_out/s3g_pytest_pf.log
timeout 600 python -m pytest tests/test_bench_contract.py -x -q -m gpu > gpurun_out/s3g_contract.log 2>&1; tail -2 gpurun_out/s3g_contract.log
REPS=6 bash scripts/gpu_ab.sh s3g C5 pf
for v in cyc pfcyc; do BM_LIB=tunelib/$v.so timeout 600 python scripts/tune.py C5 --reps 3 - > gpurun_out/s3g_$v.json 2>&1; tail -1 gpurun_out/s3g_$v.json | cut -c1-900; done
for g in tiny uniform; do BM_GRID_CTAS=1 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/racecheck_push.py $g > gpurun_out/s3g_race_$g.log 2>&1; echo "race $g rc=$?"; tail -4 gpurun_out/s3g_race_$g.log; done
