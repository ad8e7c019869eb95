cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "double_buffered" > gpurun_out/pytest_dbl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbl.log
tail -4 gpurun_out/pytest_dbl.log
