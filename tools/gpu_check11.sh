cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k model_proxy > gpurun_out/pytest_proxy.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_proxy.log
bash tools/policy_sweep.sh
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
