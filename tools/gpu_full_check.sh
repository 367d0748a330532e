# build, the GPU suite, the step timeline, one bench line
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/trace_step.py > gpurun_out/trace_step.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-bt --no-sweep --no-extra --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
