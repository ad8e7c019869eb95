cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c2 --p 0.2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2p2.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c0_full_run or tiny_slots" > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
