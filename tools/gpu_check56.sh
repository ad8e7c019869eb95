# tensor-core interleaved tile layout, one 4-D TMA per K/V segment: parity, trace, A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_cores" > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tc.log
tail -2 gpurun_out/pytest_tc.log
grep -q "pytest rc=0" gpurun_out/pytest_tc.log || exit 1
for P in 15 40 400; do
B=$((8192 * 40 / (P + 1))); [ $B -gt 8192 ] && B=8192
echo "P=$P"; timeout 300 python tools/tc_trace.py --lib tools/ab/libs3_trace.so --P $P --B $B 2>&1 | tail -1
done
echo "== new"; timeout 300 python tools/attn_sweep.py --case "tc" --custom "len16 tc:32,32,8,128,8192,15,2" --custom "len100 tc:32,32,8,128,4096,99,2" 2>&1 | grep case | cut -c1-40,150-
echo "== head"; timeout 300 python tools/attn_sweep.py --case "tc" --custom "len16 tc:32,32,8,128,8192,15,2" --custom "len100 tc:32,32,8,128,4096,99,2" --lib tools/ab/libs3_head.so 2>&1 | grep case | cut -c1-40,150-
