cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -2 gpurun_out/pytest_tc.log
for i in 1 2; do
timeout 600 python tools/attn_sweep.py --case "tc" > gpurun_out/attn_sweep_$i.log 2>&1; grep case gpurun_out/attn_sweep_$i.log
done
timeout 600 python tools/attn_sweep.py --case "mqa" > gpurun_out/attn_sweep_mqa.log 2>&1; grep case gpurun_out/attn_sweep_mqa.log
