# scratch runner for one-off GPU experiments (edited per experiment; see DESIGN §11 for results)
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/trace_step.py > gpurun_out/trace_step.log 2>&1
