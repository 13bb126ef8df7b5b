# compute-sanitizer over tools/sanitize_cases.py, one tool per invocation (B200_PROFILING.md)
tool=${1:-memcheck}
exec > gpurun_out/sanitize_$tool.log 2>&1
export SANITIZE_ELEMS=${SANITIZE_ELEMS:-3}
extra=""
[ "$tool" = "racecheck" ] && extra="--racecheck-report all"
timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py
echo "rc=$?"
