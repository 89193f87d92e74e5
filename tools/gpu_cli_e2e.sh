# the drop-in CLI end to end on a generated C5-sized Matrix Market file
mkdir -p gpurun_out
python - <<'PY'
import numpy as np, time, sys
sys.path.insert(0, ".")
from paper_2203_05096_b200 import synthetic
t = time.time()
r, c, v = synthetic.irregular_triplets(2_000_000, seed=1)
with open("/tmp/irr.mtx", "w") as fh:
    fh.write("%%MatrixMarket matrix coordinate real general\n")
    fh.write(f"2000000 2000000 {len(r)}\n")
    np.savetxt(fh, np.column_stack([r + 1, c + 1, v]), fmt="%d %d %.17g")
print("wrote", len(r), "entries in", round(time.time() - t, 1), "s")
PY
for k in cuda3 cuda35 cpu3; do
  T0=$(date +%s.%N); timeout 900 python -m paper_2203_05096_b200.cli run /tmp/irr.mtx --kernel $k --profile b200 --format json > gpurun_out/cli_$k.json 2> gpurun_out/cli_$k.err
  echo "$k wall $(echo "$(date +%s.%N) - $T0" | bc) s"; cat gpurun_out/cli_$k.json; tail -2 gpurun_out/cli_$k.err
done
