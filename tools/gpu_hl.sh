set -x
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 240 python tools/lmh_sweep.py --steady > gpurun_out/hl_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/hl_sweep.log
EVOSPEC_LMH_HL=0 timeout 240 python tools/lmh_sweep.py --n 8192,36864 > gpurun_out/old_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/old_sweep.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
