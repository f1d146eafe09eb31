# session 3: pulled-level parity with claim-time marks, then A/B (in-tree = marks; nomark; vec) on C5 and C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bottom_up or lazy or mixed or serial_retry" > gpurun_out/s3d_pytest.log 2>&1; tail -2 gpurun_out/s3d_pytest.log
BM_LIB=tunelib/vec.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "bottom_up or lazy or mixed" > gpurun_out/s3d_pytest_vec.log 2>&1; tail -2 gpurun_out/s3d_pytest_vec.log
timeout 600 python -m pytest tests/test_upload.py tests/test_full_size.py -x -q > gpurun_out/s3d_pytest2.log 2>&1; tail -2 gpurun_out/s3d_pytest2.log
REPS=6 bash scripts/gpu_ab.sh s3d C5 nomark vec
REPS=6 bash scripts/gpu_ab.sh s3d C2 nomark vec
