# usage: bash scripts/gpu_variants.sh <tag> <lib>...   stage timelines of alternative builds
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu --timeout 600 > gpurun_out/${tag}_tests.log 2>&1; tail -2 gpurun_out/${tag}_tests.log
for lib in default "$@"; do
  name=$(basename $lib .so)
  for c in C2 C3; do
    if [ "$lib" = default ]; then timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_${name}_$c.json 2>&1;
    else BM_LIB=$PWD/$lib timeout 300 python scripts/timeline.py $c > gpurun_out/${tag}_${name}_$c.json 2>&1; fi
  done
  if [ "$lib" = default ]; then timeout 300 python scripts/timeline.py C4 --div 4 > gpurun_out/${tag}_${name}_C4d4.json 2>&1;
  else BM_LIB=$PWD/$lib timeout 300 python scripts/timeline.py C4 --div 4 > gpurun_out/${tag}_${name}_C4d4.json 2>&1; fi
done
