# TC: A/B of the working tree against HEAD (tools/ab/libs3_head.so) + TC parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores or host_fed or grouped or abi_error" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -2 gpurun_out/pytest_tc.log
for i in 1 2; do
echo "== new"; timeout 200 python tools/attn_sweep.py --case "tc" 2>&1 | grep case | cut -c1-60,150-
echo "== head"; timeout 200 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case | cut -c1-60,150-
done
