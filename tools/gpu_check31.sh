# A/B on one box: HEAD's tensor-core kernel (tools/ab/libs3_head.so) vs the working tree
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1; do
echo "== head"; timeout 600 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case
echo "== new"; timeout 600 python tools/attn_sweep.py --case "tc" 2>&1 | grep case
done
