python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_oov.py -q > gpurun_out/oov_test.log 2>&1; echo "rc=$?" >> gpurun_out/oov_test.log
timeout 300 python -c "
import bench, argparse, json
a = argparse.Namespace(warmup=3, sweep_steps=5, steps=5)
print(json.dumps(bench.oov_overlap_line('cuda:0', a)))
" > gpurun_out/oov_line.log 2>&1; echo "rc=$?" >> gpurun_out/oov_line.log
