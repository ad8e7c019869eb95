# tensor-core parity for G = 3 (packed pairs), G = 8 with an odd KV-head count, G = 2 with 4 KV heads (packs of 4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "tensor_cores and (12-4 or 24-3 or 8-4)" > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g.log
grep -E "worst|passed|failed|rc=" gpurun_out/pytest_g.log | tail -6
