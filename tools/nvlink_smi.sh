#!/bin/bash
# NVLink data counters (nvidia-smi nvlink -gt d) of every GPU before and after
# a dist_steps run: the hardware's TX/RX bytes per GPU for W + K steps.
# Usage: tools/nvlink_smi.sh N N_G DENSITY STEPS OUTFILE PORT
N=$1; NG=$2; D=$3; K=$4; OUT=$5; PORT=${6:-29760}
for g in $(seq 0 $((N-1))); do nvidia-smi nvlink -gt d -i $g; done > "$OUT.before" 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
  --master-port $PORT tools/dist_steps.py --n_g $NG --density $D --warmup 0 --steps $K > "$OUT.run" 2>&1
for g in $(seq 0 $((N-1))); do nvidia-smi nvlink -gt d -i $g; done > "$OUT.after" 2>&1
