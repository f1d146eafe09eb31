#!/bin/bash
O=gpurun_out/pre1; mkdir -p $O
for v in 0 1; do
for c in C2 C1; do
BM_PREBUILD=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-alt > $O/bench_${c}_pre$v.json 2> $O/bench_${c}_pre$v.err
tail -1 $O/bench_${c}_pre$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$c pre$v', round(d['ms_per_step'],2), 'e2e', round(e['ms_per_step'],2), e.get('pulled_dense_levels'), 'pageable', round(e['pageable']['ms_per_step'],2), 'gpuinit', round(e['gpu_init']['ms_per_step'],2), d['bottom_up'])"
done; done
BM_PREBUILD=1 timeout 300 ./oracle/_ref/shim_e2e C2 10 > $O/shim_C2_pre1.json 2>&1; cat $O/shim_C2_pre1.json
