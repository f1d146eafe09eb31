# session 3 closing: smoke, GPU suite, default bench (C5), reference arm (C5), shim e2e
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/final6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.log 2>&1; tail -1 gpurun_out/final6/smoke.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/final6/pytest.log 2>&1; tail -1 gpurun_out/final6/pytest.log
timeout 1500 python bench.py > gpurun_out/final6/bench_C5.json 2> gpurun_out/final6/bench_C5.err
tail -1 gpurun_out/final6/bench_C5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['ms_per_step'],2), 'phases', d['counters_mean']['outer_iterations'], 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'], d['parity']['ok'], d['bottom_up'], d['clocks'])"
timeout 1500 python bench.py --impl reference > gpurun_out/final6/reference_C5.json 2> gpurun_out/final6/reference_C5.err
tail -1 gpurun_out/final6/reference_C5.json | cut -c1-400
timeout 900 ./oracle/_ref/shim_e2e C5 4 > gpurun_out/final6/shim_e2e_C5.json 2>&1; cat gpurun_out/final6/shim_e2e_C5.json
