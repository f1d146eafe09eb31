#!/bin/bash
O=gpurun_out/late2; mkdir -p $O
timeout 600 python scripts/late_tl.py C5 --reps 6 > $O/C5.txt 2>&1; cat $O/C5.txt | cut -c1-1500
timeout 300 python scripts/late_tl.py C2 --reps 6 BM_LATE_ROOTS=8192 > $O/C2.txt 2>&1; cat $O/C2.txt | cut -c1-1200
