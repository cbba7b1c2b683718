#!/bin/bash
# torchrun --no-python entry: run this rank under ncu with a per-rank CSV log
# (ranks listed in NCU_RANKS, default all; the others run plain).
# Usage: ncu_rank.sh OUT_PREFIX METRICS KREGEX SKIP COUNT -- cmd...
OUT=$1; METRICS=$2; KRE=$3; SKIP=$4; CNT=$5; shift 6
NCU=$(command -v ncu || echo /usr/local/cuda/bin/ncu)
R=${RANK:-0}
if [ -z "$NCU_RANKS" ] || [[ ",$NCU_RANKS," == *",$R,"* ]]; then
  exec $NCU --metrics "$METRICS" --clock-control none --cache-control none -k "regex:$KRE" \
    --launch-skip $SKIP --launch-count $CNT --csv --print-units base \
    --log-file "${OUT}_rank${R}.csv" "$@"
else
  exec "$@"
fi
