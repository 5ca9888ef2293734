# narrow-band probe on cfg4 shards
set -x
for o in "probe_ub=0" "probe_ub=1" "probe_ub=1,probe=512" "probe_ub=0,probe=512"; do OPTS=$o python tools/shard_emul.py 4 8 2>&1 | grep "N="; done
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x -k "warm_start or sharded or speculative or golden" 2>&1 | tail -3
