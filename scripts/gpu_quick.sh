# usage: bash scripts/gpu_quick.sh <tag>  — GPU tests, timelines C2/C3/C4, C2 bench (no CPU baseline)
tag=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
for c in C2 C3 C4 C1; do timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_tl_$c.json 2>gpurun_out/${tag}_tl_$c.err; tail -2 gpurun_out/${tag}_tl_$c.err; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -3 gpurun_out/${tag}_bench.err
python scripts/tl_report.py ${tag}
