cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_fed" > gpurun_out/pytest_lg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lg.log
tail -15 gpurun_out/pytest_lg.log
