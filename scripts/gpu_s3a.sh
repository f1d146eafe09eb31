# Session-3 baseline at HEAD: smoke, GPU suite (incl. slow C5), default bench (C5), MG team-of-1 C5.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3a_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a_smoke.log 2>&1; tail -1 gpurun_out/s3a_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s3a_pytest.log 2>&1; tail -2 gpurun_out/s3a_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s3a_bench.json 2> gpurun_out/s3a_bench.err; tail -c 600 gpurun_out/s3a_bench.json
timeout 900 python scripts/mg_check.py C5 > gpurun_out/s3a_mg.log 2>&1; tail -5 gpurun_out/s3a_mg.log
