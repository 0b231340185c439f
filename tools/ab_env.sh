#!/bin/bash
# Interleaved same-box A/B of one library under different environments:
#   tools/ab_env.sh "sweep args" rounds "ENV=a" "ENV=b" ...   ("-" = no override)
ARGS=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for E in "$@"; do
    echo "== $E round $r"
    if [ "$E" = "-" ]; then timeout 200 python tools/sweep.py $ARGS | cut -c1-64
    else env $E timeout 200 python tools/sweep.py $ARGS | cut -c1-64; fi
  done
done
