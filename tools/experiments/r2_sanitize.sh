# compute-sanitizer over every kernel family at tiny sizes (tools/sanitize_cases.py); TOOL = racecheck | synccheck | memcheck
mkdir -p gpurun_out
TOOL=${1:-racecheck}
EXTRA=""
[ "$TOOL" = racecheck ] && EXTRA="--racecheck-report analysis"
timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2_sanitize_$TOOL.log 2>&1; echo "exit $?"; tail -15 gpurun_out/r2_sanitize_$TOOL.log
