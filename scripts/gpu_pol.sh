tag=${1:-pol}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
timeout 1200 python scripts/policy_exp.py C2 C3 C4 C1 > gpurun_out/${tag}_pol.jsonl 2>&1; tail -2 gpurun_out/${tag}_pol.jsonl
