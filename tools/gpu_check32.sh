cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do
echo "== new mqa $i"; timeout 90 python tools/attn_sweep.py --case "mqa H=16 D=128 tc" 2>&1 | tail -3
done
echo "== head mqa"; timeout 90 python tools/attn_sweep.py --case "mqa H=16 D=128 tc" --lib tools/ab/libs3_head.so 2>&1 | tail -3
nvidia-smi --query-gpu=name,utilization.gpu --format=csv
