# session 3: level functions compiled out of line (own register allocation) — C5, C2, C4, C3
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
BM_LIB=tunelib/sweepni.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bottom_up or corpus_given" 2>&1 | tail -1
for c in C5 C2 C4 C3; do
  for v in base sweepni expandni; do
    if [ $v = base ]; then L=""; else L="tunelib/$v.so"; fi
    BM_LIB=$L timeout 900 python scripts/tune.py $c --reps 10 - > gpurun_out/s4a_${c}_$v.json 2>&1
  done
done
python - <<'PY'
import json, statistics, glob
for f in sorted(glob.glob('gpurun_out/s4a_C*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    pp = [m / p for m, p in zip(d['ms'], d['phases'])]
    print(f.split('/')[-1], 'mean %.2f' % statistics.mean(d['ms']), d['phases'], 'ms/phase %.3f' % statistics.median(pp), d['ok'])
PY
