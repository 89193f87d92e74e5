mkdir -p gpurun_out
TAG=${1:-bk}
timeout 1500 python -m pytest tests -x -q -m gpu -k "wbo or band_k or fullsize or coarsen or matching" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for i in 1 2; do timeout 300 python tools/prof_bandk_dev.py C2 > gpurun_out/bandk_prof_${i}_$TAG.txt 2>&1; done
grep -E "build|wbo-base|coarsen |expand|device" gpurun_out/bandk_prof_*_$TAG.txt
