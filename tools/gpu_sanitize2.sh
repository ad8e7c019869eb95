# compute-sanitizer over the tensor-core kernel (packed tiles, fused shift) and the host-fed step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores and (4-2-7 or 8-2-64) or host_fed_decode_step and (0-3-16 or 2-0-16)" > gpurun_out/sanitize2_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize2_$tool.log
  tail -4 gpurun_out/sanitize2_$tool.log
done
