# usage: bash scripts/gpu_final.sh <tag> — evidence for profiles/: smoke, tests, bench C2 (+CPU baseline), ncu launch list + full,
# stage timelines C1-C4, bench lines for C1, C3, C4 (no CPU baseline)
tag=${1:-final}
bash scripts/gpu_full.sh $tag
mkdir -p gpurun_out/${tag}_cubin && (cd gpurun_out/${tag}_cubin && cuobjdump -xelf all ../../paper_1303_1379_b200/libbmatch_b200.so > /dev/null)
for c in C1 C2 C3 C4; do timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_tl_$c.json 2>&1; done
for c in C1 C3 C4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$c.json 2>gpurun_out/${tag}_bench_$c.err; done
ls gpurun_out | grep $tag | head -40
