# usage: bash scripts/gpu_envab.sh <tag> "ENV=.. ENV2=.." ...  — median-of-5 per env setting (default build)
tag=$1; shift
mkdir -p gpurun_out
: > gpurun_out/${tag}_env.jsonl
for spec in "$@"; do
  echo "== $spec" >> gpurun_out/${tag}_env.jsonl
  env $spec timeout 600 python scripts/perf_exp.py C2 C3 C4 >> gpurun_out/${tag}_env.jsonl 2>>gpurun_out/${tag}_env.err
done
python -c "
import json
spec=None
for l in open('gpurun_out/${tag}_env.jsonl'):
    if l.startswith('=='): spec=l[3:].strip(); continue
    d=json.loads(l); print(spec, ' '.join(f\"{c}:{d[c]['ms_med']}ms/{d[c]['ms_per_phase']}pp/{d[c]['phases']}/{'ok' if d[c]['ok'] else 'BAD'}\" for c in ['C2','C3','C4'] if c in d))
"
tail -3 gpurun_out/${tag}_env.err
