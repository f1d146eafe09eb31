# session 3: A/B of the pulled-level probe variants (in-tree = prep, scalar probes) on C5 and C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
BM_LIB=tunelib/vechint.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bottom_up or lazy or mixed" > gpurun_out/s3e_pytest_vh.log 2>&1; tail -1 gpurun_out/s3e_pytest_vh.log
REPS=6 bash scripts/gpu_ab.sh s3e C5 vec hint vechint
REPS=6 bash scripts/gpu_ab.sh s3e C2 vec hint vechint
