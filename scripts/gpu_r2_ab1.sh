cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash scripts/gpu_ab.sh ab1 C5 cs
bash scripts/gpu_ab.sh ab1 C2 cs
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab1_c1_launches.csv python scripts/tune.py C1 --reps 1 - > gpurun_out/ab1_c1_ncu.log 2>&1; grep -c driver gpurun_out/ab1_c1_launches.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -c 1 -o gpurun_out/ab1_c5_prof python scripts/tune.py C5 --reps 0 - > gpurun_out/ab1_c5_ncu.log 2>&1; tail -3 gpurun_out/ab1_c5_ncu.log
