cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2 -c 1 -o gpurun_out/attn_tc_short python tools/attn_sweep.py --case "tc short" --steps 3 > gpurun_out/ncu_tc_short.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_tc_short.log
