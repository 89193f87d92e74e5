# one GPU pass without the (slow, CPU-only) reference arm: tests, smoke, default bench, 1-rank dist bench
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -5 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --gpus 1 --config C5 > gpurun_out/bench_C5_$TAG.json 2> gpurun_out/bench_C5_$TAG.err; echo "C5 rc=$?"
cat gpurun_out/bench_C5_$TAG.json
CSRK_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 > gpurun_out/bench_dist1_$TAG.json 2> gpurun_out/bench_dist1_$TAG.err; echo "dist1 rc=$?"
cat gpurun_out/bench_dist1_$TAG.json
