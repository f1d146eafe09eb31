set -x
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|^CPU\(s\)" ; free -g | head -2
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json
timeout 300 python bench.py --config C1 --steps 20 --warmup 3 > gpurun_out/bench_c1.json 2>&1; cat gpurun_out/bench_c1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_run.log 2>&1; tail -3 gpurun_out/ncu_launch_run.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 2 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; tail -5 gpurun_out/ncu_full.log
ls -la gpurun_out
