mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py -x -q -m gpu -k "bench_multi_gpu or native" > gpurun_out/pytest_ng.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ng.log; tail -2 gpurun_out/pytest_ng.log
for mg in native torch; do
  CSRK_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --mg $mg > gpurun_out/ng_$mg.json 2> gpurun_out/ng_$mg.err; echo "dist1 $mg rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/ng_$mg.json')); print('$mg', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['host_enqueue_us_per_step_max'], d['timed_as'], d['efficiency_t1_over_n_tn'])"
done
for mg in native torch; do
  CSRK_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --mg $mg --config C1 > gpurun_out/ng_C1_$mg.json 2> gpurun_out/ng_C1_$mg.err; echo "dist1 C1 $mg rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/ng_C1_$mg.json')); print('C1 $mg', d['ms_per_step'], d['roofline']['frac'], d['parity']['ok'], d['host_enqueue_us_per_step_max'], d['timed_as'])"
done
tail -5 gpurun_out/ng_native.err
