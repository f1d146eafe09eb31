# usage: bash scripts/gpu_part.sh <tag> — partitioned bench at N=1 (nccl) and N=2 on one GPU (gloo exchange)
tag=${1:-part}
mkdir -p gpurun_out
true
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --exchange gloo --steps 3 --warmup 3 > gpurun_out/${tag}_part2.json 2> gpurun_out/${tag}_part2.err; cat gpurun_out/${tag}_part2.json; tail -3 gpurun_out/${tag}_part2.err
