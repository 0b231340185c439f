#!/bin/bash
# ncu --set full of one ax_helm launch per lx (any kernel; on the GPU box):
#   bash tools/prof_ax.sh MODE TAG LX [LX ...]  ->  gpurun_out/TAG_l<lx>_<mode>.{ncu-rep,txt}
MODE=$1; TAG=$2; shift 2
for lx in "$@"; do
  R=gpurun_out/${TAG}_l${lx}_${MODE}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:ax_ -s 3 -c 1 -o $R -f \
    python tools/sweep.py --lx $lx --modes $MODE --reps 2 > /dev/null 2>&1
  python tools/ncu_summary.py $R.ncu-rep > $R.txt 2>&1
  python tools/ncu_lines.py $R.ncu-rep 14 >> $R.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f $R.ncu-rep  # gpurun copies back <= 64 MiB
done
