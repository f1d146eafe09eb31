#!/bin/bash
O=gpurun_out/pre2; mkdir -p $O
timeout 2000 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for c in C2 C3 C4; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-alt > $O/bench_$c.json 2> $O/bench_$c.err
tail -1 $O/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$c', round(d['ms_per_step'],2), 'e2e', round(e['ms_per_step'],2), 'pageable', round(e['pageable']['ms_per_step'],2), 'gpuinit', round(e['gpu_init']['ms_per_step'],2), d['bottom_up'])"
done
timeout 300 ./oracle/_ref/shim_e2e C2 10 > $O/shim_e2e_C2.json 2>&1; cat $O/shim_e2e_C2.json
