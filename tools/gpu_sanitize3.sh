# compute-sanitizer after the host-fed tensor-core path, mapped report and double staging
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores and (4-2-7 or 8-2-64) or host_fed_decode_step or c0_full_run or tiny_slots or sync_eviction" > gpurun_out/sanitize4_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize4_$tool.log
  tail -4 gpurun_out/sanitize4_$tool.log
done
