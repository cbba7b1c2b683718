#!/bin/bash
# NVLink TX bytes per launch of the push-reduce kernels (ncu nvltx__bytes.sum,
# one counter: a single pass, no kernel replay racing the peers). Only the rank
# in NCU_RANKS (default 1) runs under ncu: two ncu processes contend for the
# device-level NVLink counters and the second fails with UnknownError.
# Usage: tools/nvlink_ncu.sh N N_G DENSITY OUTDIR PORT
N=$1; NG=$2; D=$3; OUT=$4; PORT=${5:-29750}
mkdir -p "$OUT"
export NCU_RANKS=${NCU_RANKS:-1}
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
  --master-port $PORT --no-python \
  bash tools/ncu_rank.sh "$OUT/nvl_n${N}_${NG}_${D}" nvltx__bytes.sum,gpu__time_duration.sum \
  "exchange_kernel" 10 4 -- \
  python tools/dist_steps.py --n_g $NG --density $D --warmup 20 --steps 6 --leak
