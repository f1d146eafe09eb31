# usage: bash scripts/gpu_variants.sh <tag> <lib>...   stage timelines of alternative builds (C2, C3, C4, C1)
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
for lib in default "$@"; do
  name=$(basename $lib .so)
  for c in C2 C3 C4 C1; do
    if [ "$lib" = default ]; then timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_${name}_$c.json 2>&1;
    else BM_LIB=$PWD/$lib timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_${name}_$c.json 2>&1; fi
  done
done
python scripts/var_report.py $tag default "$@"
