mkdir -p gpurun_out
TAG=${1:-r01d}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/prof_bandk_dev.py C2 > gpurun_out/bandk_prof_eager_$TAG.txt 2>&1
grep -E "build|wbo-base|coarsen |expand|device" gpurun_out/bandk_prof_eager_$TAG.txt
CSRK_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --config C4 --steps 2 --warmup 1 --iters 100 > gpurun_out/dist_C4_$TAG.json 2> gpurun_out/dist_C4_$TAG.err
cat gpurun_out/dist_C4_$TAG.json
for C in C2 C3 C5; do timeout 600 python bench.py --config $C --steps 100 --warmup 5 --cpu-budget 2 > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; done
