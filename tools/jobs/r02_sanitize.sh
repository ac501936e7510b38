# one compute-sanitizer tool per gpurun call (B200_PROFILING.md): racecheck | memcheck | synccheck
tool=${1:-racecheck}
extra=""
[ "$tool" = racecheck ] && extra="--racecheck-report all"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 200 python tools/racecheck.py 2 3 10 20 > gpurun_out/r02_${tool}.log 2>&1; echo "$tool rc $?"
tail -12 gpurun_out/r02_${tool}.log
