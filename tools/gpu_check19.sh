cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/attn_sweep.py --case "tc" > gpurun_out/sweep_tc3.log 2>&1
S3_TC_STAGES=1 timeout 600 python tools/attn_sweep.py --case "tc" > gpurun_out/sweep_tc1.log 2>&1
S3_TC_STAGES=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores" > gpurun_out/pytest_tc1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc1.log
