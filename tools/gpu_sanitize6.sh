# memcheck after the generator changes (k_synth / k_fill) and the new tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c0_full_run or zero_length or tiny_slots or layer_group or double_buffered or host_fed_decode_step and 0-5-8" > gpurun_out/sanitize6_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize6_memcheck.log
tail -4 gpurun_out/sanitize6_memcheck.log
