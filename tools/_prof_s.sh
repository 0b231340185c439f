for lx in 12 10; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ax_line -s 3 -c 1 -o gpurun_out/r02_s2lo_l${lx}_strict -f python tools/sweep.py --lx $lx --modes strict --reps 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_s2lo_l${lx}_strict.ncu-rep > gpurun_out/r02_s2lo_l${lx}_strict.txt 2>&1
python tools/ncu_lines.py gpurun_out/r02_s2lo_l${lx}_strict.ncu-rep 14 >> gpurun_out/r02_s2lo_l${lx}_strict.txt 2>&1
done
