# session 3 checkpoint: racecheck (1-CTA grid and full grid), GPU suite, default bench (C5)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for g in tiny uniform; do BM_GRID_CTAS=1 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/racecheck_push.py $g > gpurun_out/s3h_race1_$g.log 2>&1; echo "race 1-CTA $g rc=$?"; tail -2 gpurun_out/s3h_race1_$g.log; done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/racecheck_push.py tiny > gpurun_out/s3h_racefull_tiny.log 2>&1; echo "race full tiny rc=$?"; tail -2 gpurun_out/s3h_racefull_tiny.log
BM_GRID_CTAS=1 timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_bu.py > gpurun_out/s3h_race1_bu.log 2>&1; echo "race 1-CTA bu rc=$?"; tail -2 gpurun_out/s3h_race1_bu.log
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/s3h_pytest.log 2>&1; tail -2 gpurun_out/s3h_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s3h_bench.json 2> gpurun_out/s3h_bench.err; tail -c 1500 gpurun_out/s3h_bench.json
