# late phases, check 1: smoke, GPU suite, ncu --set full of one C5 and one C2 driver_kernel, late-phase traces
cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/final7; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 2000 python -m pytest tests -q -m gpu -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python scripts/late_tl.py C5 --reps 3 > $O/late_C5.txt 2>&1; cut -c1-300 $O/late_C5.txt
for c in C5 C2; do
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:driver_kernel -s 1 -c 1 -o $O/${c}_prof python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-alt > $O/${c}_ncu.log 2>&1; tail -2 $O/${c}_ncu.log
done
ls -la $O
