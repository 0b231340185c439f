# round-1 refresh after the x-folding apply: bench line, launch list, ncu full of the folded apply and the DSSUM pass
timeout 300 python bench.py > gpurun_out/bench_s8.json 2> gpurun_out/bench_s8.err; tail -c 300 gpurun_out/bench_s8.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s8.csv python bench.py --steps 3 --warmup 3 --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_s8.csv "bench.py --steps 3 --warmup 3 --no-e2e (x-folding apply)" > gpurun_out/launches_s8.txt; head -14 gpurun_out/launches_s8.txt
timeout 400 ncu -f --set full --clock-control none --import-source on -k regex:ax_dmma8 -c 1 -o /tmp/xf python tools/axgs_run.py --reps 1 > /dev/null 2>&1
timeout 400 ncu -f --set full --clock-control none -k regex:gs_box_local_kernel -c 2 -o /tmp/gs2 python tools/axgs_run.py --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/xf.ncu-rep > gpurun_out/ncu_xf.txt 2>&1; python tools/ncu_summary.py /tmp/gs2.ncu-rep > gpurun_out/ncu_gs2.txt 2>&1
grep -E "==|duration|dram__bytes" gpurun_out/ncu_xf.txt gpurun_out/ncu_gs2.txt
