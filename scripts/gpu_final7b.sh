# late phases, check 2: bench lines C1-C5 (C5 = the default), reference arm C5, shim e2e, C5 launch list, timelines
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/final7; mkdir -p $O
timeout 1500 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
tail -1 $O/bench_C5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['ms_per_step'],2), 'phases', d['counters_mean']['outer_iterations'], 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'], d['parity']['ok'], d['roofline']['frac'], d['clocks'])"
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -1 $O/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'] if d.get('cpu_baseline') else None, d['parity']['ok'])"
done
timeout 1500 python bench.py --impl reference > $O/reference_C5.json 2> $O/reference_C5.err
tail -1 $O/reference_C5.json | cut -c1-300
timeout 900 ./oracle/_ref/shim_e2e C5 4 > $O/shim_e2e_C5.json 2>&1; cat $O/shim_e2e_C5.json
timeout 300 ./oracle/_ref/shim_e2e C2 10 > $O/shim_e2e_C2.json 2>&1; cat $O/shim_e2e_C2.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/c5_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-alt --no-e2e > $O/c5_launches_bench.log 2>&1; echo "ncu rc=$?"
for c in C2 C3 C4 C5; do timeout 600 python scripts/timeline.py $c > $O/timeline_$c.json 2>&1; done
ls $O
