import json, os, sys
tag = sys.argv[1]
for lib in sys.argv[2:]:
    name = os.path.basename(lib).replace('.so', '')
    row = [name]
    for c in ['C2', 'C3', 'C4', 'C1']:
        try:
            d = json.load(open(f'gpurun_out/{tag}_{name}_{c}.json'))
            row.append(f"{c}:{d['kernel_ms']:.2f}ms/{d['n_phases']}ph/{d['n_levels']}lv{'' if d['known'] in (None, d['cardinality']) else ' BAD'}")
        except Exception as e:
            row.append(f"{c}:ERR")
    print('  '.join(row))
