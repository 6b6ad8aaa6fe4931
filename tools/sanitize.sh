#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_run.py.
#   tools/sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck synccheck racecheck initcheck; do
  ARGS="--small"
  EXTRA=""
  [ "$T" = "memcheck" ] && EXTRA="--leak-check no"
  [ "$T" = "racecheck" ] && EXTRA="--racecheck-report all"
  timeout 900 $CS --tool $T $EXTRA --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py $ARGS \
    > gpurun_out/${TAG}_${T}.log 2>&1
  echo "$T exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done" gpurun_out/${TAG}_${T}.log | tail -3
done
