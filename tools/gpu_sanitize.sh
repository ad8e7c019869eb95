cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -x -k "poison or zero_length" > gpurun_out/pytest_gpu_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_new.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c0_full_run or zero_length or tiny_slots" > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
