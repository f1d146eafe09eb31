#!/bin/bash
# Round-2 check on one B200: GPU tests (incl. C5), the default bench line (C5)
# and the reference arm as the driver runs them.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
nproc >> gpurun_out/r2_smi.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} ) > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
if [ -z "$SKIP_BENCH" ]; then
( time timeout 900 python bench.py --steps 10 --warmup 3 ) > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
fi
tail -3 gpurun_out/r2_pytest.log
