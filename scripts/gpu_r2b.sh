cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -x -q -m gpu -k "bottom_up or pulled or full_size or retry" > gpurun_out/r2b_pytest.log 2>&1; tail -3 gpurun_out/r2b_pytest.log
timeout 900 python scripts/tune.py C5 --tl - > gpurun_out/r2b_tune_c5.json 2>&1
timeout 900 python scripts/tune.py C5 BM_BU_ALPHA=4 BM_BU_ALPHA=8 BM_BU_ALPHA=30 BM_BU_ALPHA=60 BM_BU_FRAC=0.2 BM_BU_FRAC=0.05 BM_PAIRS_MIN_EDGES=999999999999 >> gpurun_out/r2b_tune_c5.json 2>&1
timeout 600 python scripts/tune.py C2 --tl - BM_BU_ALPHA=2 BM_BU_ALPHA=8 BM_BU_ALPHA=14 BM_BU_FRAC=0.45 TUNE_BU=off > gpurun_out/r2b_tune_c2.json 2>&1
