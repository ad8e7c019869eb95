# per-role timeline of the tensor-core kernel (diagnostic TC_TRACE build)
cd $GRAFT_REPO_ROOT
for P in 15 40 100 400; do
B=$((8192 * 40 / (P + 1))); [ $B -gt 8192 ] && B=8192
echo "P=$P B=$B"; timeout 300 python tools/tc_trace.py --lib tools/ab/libs3_trace.so --P $P --B $B 2>&1 | tail -1
done
