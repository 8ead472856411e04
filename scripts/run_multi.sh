#!/bin/bash
# Launch bench.py on N GPUs of one node (one process per GPU, NCCL over NVLink), the way the
# driver's scaling run does.  usage: scripts/run_multi.sh N [bench.py args...]
#   scripts/run_multi.sh 8 --config C5 --steps 3 --warmup 3            # database-sharded (default)
#   scripts/run_multi.sh 8 --config C5 --shard queries                 # query-sharded comparison
set -e
N=${1:-8}; shift || true
PORT=${MASTER_PORT:-29517}
exec python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
    --master-port "$PORT" "$(dirname "$0")/../bench.py" --gpus "$N" "$@"
