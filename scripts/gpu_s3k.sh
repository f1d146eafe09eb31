# session 3: random-access ceilings (ubench at the C5 table sizes), C2 bench line (pageable e2e), MG C2 timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ./scripts/ubench_gather > gpurun_out/s3k_ubench.txt 2>&1; tail -3 gpurun_out/s3k_ubench.txt
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/s3k_c2_bench.json 2> gpurun_out/s3k_c2_bench.err; tail -c 800 gpurun_out/s3k_c2_bench.json
timeout 600 python scripts/mg_check.py C2 > gpurun_out/s3k_mg_c2.log 2>&1; tail -5 gpurun_out/s3k_mg_c2.log
