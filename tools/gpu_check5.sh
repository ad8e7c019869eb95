cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -x -k "layer_group or error_codes" > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu5.log
timeout 900 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c1.log
timeout 900 python bench.py --config c2 --p 0.1 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c2.log
timeout 900 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3.log
timeout 300 python bench.py --impl reference --steps 20 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
