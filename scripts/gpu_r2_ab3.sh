cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -x -q -m gpu > gpurun_out/ab3_pytest.log 2>&1; tail -3 gpurun_out/ab3_pytest.log
REPS=6 bash scripts/gpu_ab.sh ab3 C5 old minb3
REPS=6 bash scripts/gpu_ab.sh ab3 C2 old minb3
