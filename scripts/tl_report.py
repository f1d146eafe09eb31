import json, sys
tag = sys.argv[1]
for f in ['C2', 'C3', 'C4', 'C1']:
    try:
        d = json.load(open(f'gpurun_out/{tag}_tl_{f}.json'))
    except Exception:
        try: print(f, 'ERR', open(f'gpurun_out/{tag}_tl_{f}.json').read()[-1500:])
        except Exception: pass
        continue
    print(f, 'kernel_ms', round(d['kernel_ms'], 2), {k: round(v) for k, v in d['per_kind_us'].items()}, 'levels', d['n_levels'], 'phases', d['n_phases'], 'card', d['cardinality'], d['known'])
    print('  launches/phase', d['launches_per_phase'])
    print('  counters', d['counters'])
    print('  levels', d['levels_us'][:24])
try:
    b = json.load(open(f'gpurun_out/{tag}_bench.json'))
    print('bench', b['config']['workload'][:3], 'ms', round(b['ms_per_step'], 2), 'frac', round(b['roofline']['frac'], 4), 'e2e ms', b['e2e'] and round(b['e2e']['ms_per_step'], 1), 'cpu s', b['cpu_baseline'] and b['cpu_baseline']['seconds'], 'parity', b['parity'])
except Exception as e:
    print('bench ERR', e)
