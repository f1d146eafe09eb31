# usage: bash scripts/gpu_tl.sh <tag>  — GPU tests, stage timelines, C2 bench, optional ncu (NCU=1)
tag=${1:-tl}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -3 gpurun_out/${tag}_tests.log
for c in C2 C3 C1; do timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_tl_$c.json 2>gpurun_out/${tag}_tl_$c.err; tail -2 gpurun_out/${tag}_tl_$c.err; done
timeout 300 python scripts/timeline.py C4 --div 4 > gpurun_out/${tag}_tl_C4d4.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; tail -2 gpurun_out/${tag}_bench_c2.err
if [ "${NCU:-0}" = "1" ]; then
  mkdir -p gpurun_out/${tag}_cubin && (cd gpurun_out/${tag}_cubin && cuobjdump -xelf all ../../paper_1303_1379_b200/libbmatch_b200.so > /dev/null)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 2 -c 1 -o gpurun_out/${tag}_prof_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu.log 2>&1; tail -1 gpurun_out/${tag}_ncu.log
fi
