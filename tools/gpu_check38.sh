cd $GRAFT_REPO_ROOT
for i in 1; do
echo "== new"; timeout 200 python tools/attn_sweep.py --case "tc" 2>&1 | grep case | cut -c1-60,150-
echo "== head"; timeout 200 python tools/attn_sweep.py --case "tc" --lib tools/ab/libs3_head.so 2>&1 | grep case | cut -c1-60,150-
done
