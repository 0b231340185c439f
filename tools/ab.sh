#!/bin/bash
# A/B of two library builds on the same box, interleaved: tools/ab.sh A.so B.so "sweep args" [rounds]
A=$1; B=$2; ARGS=$3; R=${4:-2}
for r in $(seq 1 $R); do
  echo "== A round $r"; AXHELM_LIB=$A timeout 200 python tools/sweep.py $ARGS | cut -c1-64
  echo "== B round $r"; AXHELM_LIB=$B timeout 200 python tools/sweep.py $ARGS | cut -c1-64
done
