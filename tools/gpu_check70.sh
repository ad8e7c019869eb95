# final checks of the 4-D + ping-pong tensor-core kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/f4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f4_pytest.log
tail -n 2 gpurun_out/f4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f4_smoke.log; tail -n 1 gpurun_out/f4_smoke.log
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores and (4-2-7 or 8-2-64 or 16-1-128) or host_fed_decode_step and 2-0-16 or layer_group" > gpurun_out/f4_sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/f4_sanitize_$tool.log
  tail -n 3 gpurun_out/f4_sanitize_$tool.log
done
timeout 300 python tools/attn_sweep.py --case "tc" > gpurun_out/f4_sweep.log 2>&1; grep case gpurun_out/f4_sweep.log | cut -c1-40,150-
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/f4_tc_short python tools/attn_sweep.py --case "tc short" --steps 3 > gpurun_out/f4_ncu1.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/f4_tc_gqa python tools/attn_sweep.py --case "llama3-8b gqa tc" --steps 3 > gpurun_out/f4_ncu2.log 2>&1; echo "rc=$?"
