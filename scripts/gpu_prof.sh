# usage: bash scripts/gpu_prof.sh <tag> [config]  — ncu --set full of one driver_kernel run (+ cubin for source mapping)
tag=${1:-prof}; cfg=${2:-C2}
mkdir -p gpurun_out/${tag}_cubin && (cd gpurun_out/${tag}_cubin && cuobjdump -xelf all ../../paper_1303_1379_b200/libbmatch_b200.so > /dev/null)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 2 -c 1 -o gpurun_out/${tag}_prof python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu.log 2>&1; tail -2 gpurun_out/${tag}_ncu.log
