# usage: bash scripts/gpu_ab.sh <tag> <cfg> <variant>...  — tune.py A/B of tunelib/<variant>.so against the in-tree build
tag=$1; cfg=$2; shift 2
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python scripts/tune.py $cfg --tl --reps ${REPS:-4} - > gpurun_out/${tag}_${cfg}_base.json 2>&1
for v in "$@"; do
  BM_LIB=tunelib/$v.so timeout 600 python scripts/tune.py $cfg --tl --reps ${REPS:-4} - > gpurun_out/${tag}_${cfg}_$v.json 2>&1
done
for f in gpurun_out/${tag}_${cfg}_*.json; do echo "$f"; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('ms_min','ms_med','ms','phases','ok','edges_traversed')})"; done
