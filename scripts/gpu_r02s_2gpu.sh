#!/usr/bin/env bash
# round 2: sharded search scaling at B = 10^4 and 10^5 (1 vs 2 GPUs)
cd "$(dirname "$0")/.."
O=gpurun_out
for cfg in "c4 10000" "c4 100000" "c2 100000"; do
  set -- $cfg
  timeout 600 python scripts/dist_scale.py $1 $2 1 3 >> $O/r02s_scale.jsonl 2>> $O/r02s_scale.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29541 scripts/dist_scale.py $1 $2 1 3 >> $O/r02s_scale.jsonl 2>> $O/r02s_scale.err
done
