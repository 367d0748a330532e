set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lmh_finalize32" -s 2 -c 1 -o gpurun_out/prof9 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu9.log 2>&1
