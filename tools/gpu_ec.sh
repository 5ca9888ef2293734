# A/B: EC part of the cumulative-bound thresholds from strip 1 / 2 / 3
set -x
for rep in 1 2; do
  for o in "cb_ec_strip=1" "cb_ec_strip=2" "cb_ec_strip=3" "cb_ec_strip=5"; do
    OPTS=$o python tools/plan_timing.py bisect_libs/lib_ec.so 2>&1 | tail -1
  done
done
for c in cfg3 cfg2; do for o in "cb_ec_strip=1" "cb_ec_strip=2"; do CFG=$c OPTS=$o python tools/plan_timing.py bisect_libs/lib_ec.so 2>&1 | tail -1; done; done
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "baseline or tighten or fp32 or golden or variant" 2>&1 | tail -3
