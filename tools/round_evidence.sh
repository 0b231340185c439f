#!/bin/bash
# End-of-session evidence on one B200 (run under gpurun):
#   bash tools/round_evidence.sh TAG
# -> gpurun_out/TAG_{gpu_tests,smoke}.txt, TAG_bench.json (default bench line),
#    TAG_launches.{csv,txt} (ncu launch list of a short bench), TAG_ncu_dmma8.txt
#    (ncu --set full of the headline kernel at C2)
T=${1:-rXX}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $O/${T}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/${T}_gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --gs-steps 2 --cg-iters 3 --c4-steps 2 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
python tools/launch_summary.py $O/${T}_launches.csv \
  "ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 3 --gs-steps 2 --cg-iters 3 --c4-steps 2 --no-e2e --no-cpu --no-sweep" \
  > $O/${T}_launches.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ax_dmma8 -s 3 -c 1 -o $O/${T}_dmma8 -f \
  python tools/sweep.py --lx 8 --points 134217728 --modes fast --reps 2 > /dev/null 2>&1
python tools/ncu_summary.py $O/${T}_dmma8.ncu-rep > $O/${T}_ncu_dmma8.txt 2>&1
rm -f $O/${T}_dmma8.ncu-rep
tail -3 $O/${T}_gpu_tests.txt; cat $O/${T}_smoke.txt; head -c 700 $O/${T}_bench.json; echo; head -12 $O/${T}_launches.txt; head -6 $O/${T}_ncu_dmma8.txt
