python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "lmh_paths or medium" > gpurun_out/gemv_test.log 2>&1; echo "rc=$?" >> gpurun_out/gemv_test.log
timeout 300 python -c "
import bench, argparse, json, torch, numpy as np, synth
import paper_2605_27390_b200 as es
a = argparse.Namespace(warmup=3, sweep_steps=10, steps=5)
c = dict(synth.CONFIGS['llama']); V, d = c['V'], c['d']
bf = torch.bfloat16
W = torch.from_numpy(synth.matrix(0, V, d, 0.02, 'bf16').view(np.int16)).view(bf).cuda()
H = torch.from_numpy(synth.matrix(1, 60, d, 1.0, 'bf16').view(np.int16)).view(bf).cuda()
ctx = es.Context(V=V, d=d, w_dtype=bf, h_dtype=bf, max_subset=V, max_rows=60, max_k=10)
ctx.prepare_weights(W)
print(json.dumps(bench.per_depth_line(ctx, W, H, 10, V, d, 'cuda:0', a)))
" > gpurun_out/gemv_line.log 2>&1
