# usage: bash scripts/gpu_explore.sh <tag>  — stage timelines for C1-C4 and the WR claim-policy experiment
tag=${1:-ex}
mkdir -p gpurun_out
for c in C2 C3 C1 C4; do timeout 400 python scripts/timeline.py $c > gpurun_out/${tag}_tl_$c.json 2>gpurun_out/${tag}_tl_$c.err; tail -2 gpurun_out/${tag}_tl_$c.err; done
timeout 400 python scripts/timeline.py C2 apsb-wr > gpurun_out/${tag}_tl_C2apsb.json 2>&1
timeout 900 python scripts/claim_exp.py > gpurun_out/${tag}_claim.jsonl 2>&1; tail -3 gpurun_out/${tag}_claim.jsonl
