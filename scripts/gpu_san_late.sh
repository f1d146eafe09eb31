#!/bin/bash
O=gpurun_out/san_late; mkdir -p $O
timeout 900 python scripts/sanitize_late.py > $O/plain.log 2>&1; tail -2 $O/plain.log
for t in memcheck racecheck synccheck; do
timeout 1500 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_late.py > $O/$t.log 2>&1; echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|late sanitize" $O/$t.log | tail -3
done
