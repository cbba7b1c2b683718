#!/bin/bash
# NVLink bytes per launch of the push-reduce kernels, from ncu's NVLink
# counters, on N ranks (one ncu per rank; single-pass metrics so no kernel
# replay races the peers). Usage: tools/nvlink_ncu.sh N N_G DENSITY OUTDIR PORT
N=$1; NG=$2; D=$3; OUT=$4; PORT=${5:-29750}
mkdir -p "$OUT"
NCU=$(command -v ncu || echo /usr/local/cuda/bin/ncu)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
  --master-port $PORT --no-python \
  $NCU --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum \
  --clock-control none --cache-control none -k "regex:stream_kernel|exchange_kernel" \
  --launch-skip 60 --launch-count 6 --csv --print-units base \
  --log-file "$OUT/nvl_n${N}_${NG}_${D}_rank%q{RANK}.csv" \
  python tools/dist_steps.py --n_g $NG --density $D --warmup 40 --steps 4
