timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmh_hl -s 2 -c 1 -o gpurun_out/prof_hl_36k python tools/lmh_sweep.py --n 36864 --iters 2 > gpurun_out/ncu_hl.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_hl.log
