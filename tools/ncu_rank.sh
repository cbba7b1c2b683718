#!/bin/bash
# torchrun --no-python entry: rank 0 runs under ncu (per-rank log file), the
# other ranks run plain. Usage: ncu_rank.sh OUT_PREFIX METRICS KREGEX SKIP COUNT -- cmd...
OUT=$1; METRICS=$2; KRE=$3; SKIP=$4; CNT=$5; shift 6
NCU=$(command -v ncu || echo /usr/local/cuda/bin/ncu)
if [ "${RANK:-0}" = "0" ]; then
  exec $NCU --metrics "$METRICS" --clock-control none --cache-control none -k "regex:$KRE" \
    --launch-skip $SKIP --launch-count $CNT --csv --print-units base \
    --log-file "${OUT}_rank0.csv" "$@"
else
  exec "$@"
fi
