# usage: bash scripts/gpu_perf.sh <tag> <lib|default>[:persistMB] ...  — median-of-5 A/B of builds
tag=$1; shift
mkdir -p gpurun_out
: > gpurun_out/${tag}_perf.jsonl
for spec in "$@"; do
  lib=${spec%%:*}; pm=0; [ "$spec" != "$lib" ] && pm=${spec#*:}
  if [ "$lib" = default ]; then BM_PERSIST_MB=$pm timeout 400 python scripts/perf_exp.py C2 C3 C4 >> gpurun_out/${tag}_perf.jsonl 2>gpurun_out/${tag}_perf.err;
  else BM_LIB=$PWD/$lib BM_PERSIST_MB=$pm timeout 400 python scripts/perf_exp.py C2 C3 C4 >> gpurun_out/${tag}_perf.jsonl 2>>gpurun_out/${tag}_perf.err; fi
done
python -c "
import json
for l in open('gpurun_out/${tag}_perf.jsonl'):
    d=json.loads(l); print(d['lib'], 'persist', d['persist'], ' '.join(f\"{c}:{d[c]['ms_med']}ms/{d[c]['ms_per_phase']}pp/{'ok' if d[c]['ok'] else 'BAD'}\" for c in ['C2','C3','C4'] if c in d))
"
grep -h "persisting" gpurun_out/${tag}_perf.err | sort | uniq
