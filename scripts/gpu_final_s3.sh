# session 3 final measurements: smoke, bench lines C1-C5 (C5 = the default, 20 steps), the C5 launch list
# (ncu gpu__time_duration, cold-cache serialised), stage timelines C2-C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out/final4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4/smoke.log 2>&1; tail -1 gpurun_out/final4/smoke.log
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final4/bench_$c.json 2> gpurun_out/final4/bench_$c.err
  tail -1 gpurun_out/final4/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'] if d.get('cpu_baseline') else None, d['parity']['ok'])"
done
timeout 1500 python bench.py > gpurun_out/final4/bench_C5.json 2> gpurun_out/final4/bench_C5.err
tail -1 gpurun_out/final4/bench_C5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'], d['parity']['ok'])"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/final4/c5_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-alt --no-e2e > gpurun_out/final4/c5_launches_bench.log 2>&1; echo "ncu rc=$?"
for c in C2 C3 C4 C5; do timeout 600 python scripts/timeline.py $c > gpurun_out/final4/timeline_$c.json 2>&1; done
ls gpurun_out/final
