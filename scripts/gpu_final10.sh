# closing measurements, last build (tuned late bounds): ncu (traffic), smoke, GPU suite, bench C1-C5, reference C5, shim e2e, launches, timelines
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/final10; mkdir -p $O
for c in C5 C2; do
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 1 -c 1 -o $O/${c}_prof python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-alt > $O/${c}_ncu.log 2>&1
python scripts/ncu_traffic.py $O/${c}_prof.ncu-rep $c final10 > $O/${c}_traffic.json 2>&1; cat $O/${c}_traffic.json | cut -c1-300
python scripts/ncu_summary.py $O/${c}_prof.ncu-rep > $O/${c}_ncu_summary.json 2>&1
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 2000 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 1500 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
tail -1 $O/bench_C5.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', round(d['ms_per_step'],2), 'phases', d['counters_mean']['outer_iterations'], 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'], d['parity']['ok'], d['roofline']['frac'], d['roofline']['traffic'], d['clocks'])"
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  tail -1 $O/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'cpu', d['cpu_baseline']['seconds'] if d.get('cpu_baseline') else None, d['parity']['ok'])"
done
timeout 1500 python bench.py --impl reference > $O/reference_C5.json 2> $O/reference_C5.err
tail -1 $O/reference_C5.json | cut -c1-300
timeout 900 ./oracle/_ref/shim_e2e C5 4 > $O/shim_e2e_C5.json 2>&1; cat $O/shim_e2e_C5.json
timeout 300 ./oracle/_ref/shim_e2e C2 10 > $O/shim_e2e_C2.json 2>&1; cat $O/shim_e2e_C2.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/c5_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-alt --no-e2e > $O/c5_launches_bench.log 2>&1; echo "ncu rc=$?"
for c in C2 C5; do timeout 600 python scripts/timeline.py $c > $O/timeline_$c.json 2>&1; done
timeout 300 python scripts/late_tl.py C5 --reps 2 > $O/late_C5.txt 2>&1
ls $O | wc -l
