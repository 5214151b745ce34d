# usage (GPU box): bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck
# one compute-sanitizer tool per gpurun call (B200_PROFILING.md); small cases only
T=$1
timeout 1500 compute-sanitizer --tool $T --print-limit 50 --log-file gpurun_out/r02_sanitize_$T.log \
  python tools/sanitize_cases.py > gpurun_out/r02_sanitize_$T.out 2>&1
echo "exit $?" >> gpurun_out/r02_sanitize_$T.out
tail -5 gpurun_out/r02_sanitize_$T.out; tail -20 gpurun_out/r02_sanitize_$T.log
