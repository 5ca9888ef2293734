# rank pass on / off on cfg4 shards (where does the warm start stop paying?)
set -x
for o in "" "rank_stride=0"; do OPTS=$o python tools/shard_emul.py 2 4 8 16 2>&1 | grep "N="; done
