for e in "X=1" "CSRK_LONG_BESIDE_NX=8"; do
  echo "== $e"
  env $e timeout 600 python tools/powerlaw_probe.py 2000000 1000 20000 2>&1 | grep -v "^\[bench"
done
