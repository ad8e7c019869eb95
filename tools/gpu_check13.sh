cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.log 2>&1
