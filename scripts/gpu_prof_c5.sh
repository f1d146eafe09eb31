# usage: bash scripts/gpu_prof_c5.sh <tag>  — C5 device timeline (tune.py --tl) + ncu capture of one C5 driver_kernel
tag=${1:-c5prof}
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/tune.py C5 --tl --reps 3 - > gpurun_out/${tag}_tune.json 2> gpurun_out/${tag}_tune.err
tail -c 600 gpurun_out/${tag}_tune.json
if [ "${NCU:-1}" = "1" ]; then
mkdir -p gpurun_out/${tag}_cubin && (cd gpurun_out/${tag}_cubin && cuobjdump -xelf all ../../paper_1303_1379_b200/libbmatch_b200.so > /dev/null)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 1 -c 1 -o gpurun_out/${tag}_prof python bench.py --config C5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-alt > gpurun_out/${tag}_ncu.log 2>&1; tail -3 gpurun_out/${tag}_ncu.log
fi
