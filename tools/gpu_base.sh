set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_base.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_base.log
