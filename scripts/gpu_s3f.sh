# session 3: pulled-sweep cycle split (cyc build), probe width A/B, pull-rule alpha sweep on C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
BM_LIB=tunelib/cyc.so timeout 600 python scripts/tune.py C5 --reps 3 - > gpurun_out/s3f_cyc.json 2>&1; tail -1 gpurun_out/s3f_cyc.json | cut -c1-1500
REPS=5 bash scripts/gpu_ab.sh s3f C5 probe2 probe8
timeout 900 python scripts/tune.py C5 --reps 4 BM_BU_ALPHA=6 BM_BU_ALPHA=10 BM_BU_ALPHA=20 BM_BU_ALPHA=30 > gpurun_out/s3f_alpha.json 2>&1; cat gpurun_out/s3f_alpha.json | cut -c1-300
