for sr in 128 96 64 48; do echo "segrows=$sr"; EVOSPEC_SEG_ROWS=$sr python tools/bench_bt.py 2>&1 | grep -E "ragged Bt|static only|dyn only"; done > gpurun_out/segrows.log 2>&1
