# ncu --set full of the default-path attention kernel (fused attend-and-shift), current code
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_attn_tma -s 20 -c 1 -o gpurun_out/attn_tma_c1_final python bench.py --steps 25 --warmup 3 --no-e2e --no-cpu-baseline --arena-gb 40 > gpurun_out/ncu_attn_tma_final.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_attn_tma_final.log
tail -3 gpurun_out/ncu_attn_tma_final.log
ls -la gpurun_out/
