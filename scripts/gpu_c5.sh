# usage: bash scripts/gpu_c5.sh <tag> <lib>...  — C5 (1.6e9 edges) median-of-5 per build
tag=$1; shift
mkdir -p gpurun_out
free -g | head -2
for l in "$@"; do BM_LIB=$PWD/$l timeout 1500 python scripts/perf_exp.py C5 >> gpurun_out/${tag}_c5.jsonl 2>>gpurun_out/${tag}_c5.err; done
cat gpurun_out/${tag}_c5.jsonl; tail -3 gpurun_out/${tag}_c5.err
