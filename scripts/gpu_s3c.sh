# session 3: C5 ncu --set full of the timed driver kernel + GPU tests of the upload path
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_upload.py -x -q > gpurun_out/s3c_upload.log 2>&1; tail -3 gpurun_out/s3c_upload.log
NCU=1 bash scripts/gpu_prof_c5.sh s3c5n 2>&1 | tail -3
