python -c "import __graft_entry__ as g; g.build()" || exit 1
for k in "multitile and 10-False" "multitile and 1-False"; do
  timeout 900 compute-sanitizer --tool racecheck python -m pytest tests -m gpu -q -x -k "$k" > gpurun_out/rc.log 2>&1
  echo "[$k] $(grep 'RACECHECK SUMMARY' gpurun_out/rc.log) $(grep -c 'sem.cu' gpurun_out/rc.log) $(tail -1 gpurun_out/rc.log)"
done
EVOSPEC_SCAN_IL=0 timeout 900 compute-sanitizer --tool racecheck python -m pytest tests -m gpu -q -x -k "multitile and 10-False" > gpurun_out/rc.log 2>&1; echo "[il0] $(grep 'RACECHECK SUMMARY' gpurun_out/rc.log)"
AB_VARIANTS="new" bash tools/gpu_ab.sh
