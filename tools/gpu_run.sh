#!/usr/bin/env bash
# One parameterised runner for the GPU-box recipes whose outputs are kept in
# profiles/ (replaces round 1's per-lease gpu_check*.sh / gpu_sanitize*.sh).
#
#   gpurun --timeout T -- 'bash tools/gpu_run.sh RECIPE TAG [args...]'
#
# recipes (outputs land in gpurun_out/TAG.*):
#   pytest   TAG [pytest -k expr]        the -m gpu suite (optionally filtered)
#   bench    TAG [bench.py args]         one bench line (JSON in TAG.json)
#   launches TAG [bench.py args]         ncu launch list (time + DRAM bytes per launch) of a bench command
#   full     TAG KREGEX SKIP [bench args]  ncu --set full of one launch of kernel KREGEX after SKIP launches
#   sanitize TAG TOOL [pytest -k expr]   compute-sanitizer (memcheck|synccheck|racecheck) over GPU tests
#   sweep    TAG [attn_sweep.py args]    tools/attn_sweep.py
#   sass     TAG                         SASS census of libs3.so (tcgen05 / TMA / bulk-copy mnemonics)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
recipe=$1; tag=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > "gpurun_out/$tag.build.log" 2>&1
case "$recipe" in
  pytest)
    if [ $# -gt 0 ]; then k=(-k "$*"); else k=(); fi
    timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider "${k[@]}" > "gpurun_out/$tag.log" 2>&1
    echo "rc=$?" >> "gpurun_out/$tag.log"; tail -3 "gpurun_out/$tag.log" ;;
  bench)
    timeout 1500 python bench.py "$@" > "gpurun_out/$tag.json" 2> "gpurun_out/$tag.err"
    echo "rc=$?"; tail -c 600 "gpurun_out/$tag.json" ;;
  launches)
    timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file "gpurun_out/$tag.csv" python bench.py "$@" > "gpurun_out/$tag.log" 2>&1
    echo "rc=$?" >> "gpurun_out/$tag.log"; tail -2 "gpurun_out/$tag.log" ;;
  full)
    kre=$1; skip=$2; shift 2
    timeout 2400 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 1 \
      -o "gpurun_out/$tag" python bench.py "$@" > "gpurun_out/$tag.log" 2>&1
    echo "rc=$?" >> "gpurun_out/$tag.log"
    ncu -i "gpurun_out/$tag.ncu-rep" --page raw --csv > "gpurun_out/${tag}_raw.csv" 2>/dev/null
    tail -2 "gpurun_out/$tag.log" ;;
  sanitize)
    tool=$1; shift
    if [ $# -gt 0 ]; then k=(-k "$*"); else k=(); fi
    timeout 2400 compute-sanitizer --tool "$tool" --target-processes all --print-limit 20 \
      python -m pytest tests -m gpu -q -x -p no:cacheprovider "${k[@]}" > "gpurun_out/$tag.log" 2>&1
    echo "rc=$?" >> "gpurun_out/$tag.log"; tail -4 "gpurun_out/$tag.log" ;;
  sweep)
    timeout 1500 python tools/attn_sweep.py "$@" > "gpurun_out/$tag.log" 2>&1
    echo "rc=$?" >> "gpurun_out/$tag.log"; tail -5 "gpurun_out/$tag.log" ;;
  sass)
    python tools/sass_census.py > "gpurun_out/$tag.txt"; cat "gpurun_out/$tag.txt" ;;
  *) echo "unknown recipe $recipe"; exit 2 ;;
esac
