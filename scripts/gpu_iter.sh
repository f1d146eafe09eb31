# usage: bash scripts/gpu_iter.sh <tag>   (tests, C2 bench, ncu full capture of the driver kernel)
tag=${1:-iter}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -5 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench_c2.err; cat gpurun_out/${tag}_bench_c2.json; tail -3 gpurun_out/${tag}_bench_c2.err
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 2 -c 1 -o gpurun_out/${tag}_prof_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_full.log 2>&1; tail -2 gpurun_out/${tag}_ncu_full.log
fi
