# one-GPU checks of the multi-GPU paths (torchrun with one rank, NCCL up)
mkdir -p gpurun_out
TAG=${1:-dist1}
CSRK_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/dist_C2_$TAG.json 2> gpurun_out/dist_C2_$TAG.err; echo "rc=$?" >> gpurun_out/dist_C2_$TAG.err
CSRK_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --config C4 --steps 2 --warmup 1 --iters 100 > gpurun_out/dist_C4_$TAG.json 2> gpurun_out/dist_C4_$TAG.err; echo "rc=$?" >> gpurun_out/dist_C4_$TAG.err
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --iters 100 > gpurun_out/C4_$TAG.json 2> gpurun_out/C4_$TAG.err
cat gpurun_out/dist_C2_$TAG.json gpurun_out/dist_C4_$TAG.json gpurun_out/C4_$TAG.json
tail -3 gpurun_out/dist_C2_$TAG.err gpurun_out/dist_C4_$TAG.err
for i in 1 2; do timeout 300 python tools/prof_bandk_dev.py C2 > gpurun_out/bandk_prof_${i}_$TAG.txt 2>&1; done
tail -5 gpurun_out/bandk_prof_1_$TAG.txt
