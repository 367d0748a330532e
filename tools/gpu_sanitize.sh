# compute-sanitizer memcheck over the GPU suite minus the full-size cases (which take too long
# under the sanitizer), racecheck / synccheck over the kernels added this session on small cases
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests -m gpu -q -x -k "not full_size and not qwen and not llama and not batched_full and not full_vocab and not sharded" > gpurun_out/sanitizer_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck.log
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest tests -m gpu -q -x -k "odd_shapes or test_kd_loss or coverage or subset_update and random or multitile and 10-False or tiny or ragged_lmh or merged or ties_tiles or two_list_integer" > gpurun_out/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck.log
timeout 1800 compute-sanitizer --tool synccheck --error-exitcode 99 python -m pytest tests -m gpu -q -x -k "odd_shapes or test_kd_loss or coverage_edges or multitile and 10-False" > gpurun_out/sanitizer_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_synccheck.log
tail -4 gpurun_out/sanitizer_memcheck.log gpurun_out/sanitizer_racecheck.log gpurun_out/sanitizer_synccheck.log
