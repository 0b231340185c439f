#!/bin/bash
# Interleaved same-box A/B of several library builds:
#   tools/abn.sh "sweep args" rounds lib1.so lib2.so ...
ARGS=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for L in "$@"; do
    echo "== $L round $r"; AXHELM_LIB=$L timeout 200 python tools/sweep.py $ARGS | cut -c1-64
  done
done
