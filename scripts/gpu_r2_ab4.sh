cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in C2 C3 C4 C5; do REPS=6 bash scripts/gpu_ab.sh ab4 $c minb3 minb2 m3i8 m3cs m3p8 > /dev/null 2>&1; done
python - <<'PY'
import json,glob,statistics
for f in sorted(glob.glob('gpurun_out/ab4_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    pp=[m/p for m,p in zip(d['ms'],d['phases'])]
    print(f, 'ms med %.2f  ms/phase med %.3f min %.3f'%(d['ms_med'], statistics.median(pp),min(pp)), d['phases'], d['ok'])
PY
