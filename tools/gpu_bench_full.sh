# round-end evidence: full bench line, reference arm, launch list, ncu --set full of the step's kernels,
# step timeline, the GPU suite
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r02.log
timeout 300 python tools/trace_step.py > gpurun_out/trace_step_r02.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --no-bt --no-extra > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sem_scan|topn_cand|union_kernel|lmh_tc|lmh_fin64|static_bits" -s 8 -c 6 -o gpurun_out/prof_r02_step -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-bt --no-extra --no-sweep > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
