cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/repro_c3.py C3 8 - BM_BU_FRAC=1.0,BM_SOLO_EDGES=0 BM_CHECK=1 > gpurun_out/r2c_c3.log 2>&1
tail -8 gpurun_out/r2c_c3.log
