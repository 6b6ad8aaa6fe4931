#!/bin/bash
# ncu --set full captures (with source) of the named kernels of one config-2 sweep.
#   tools/ncu_capture.sh TAG "regex1 regex2 ..." [config]
TAG=$1; CFG=${3:-2}
mkdir -p gpurun_out
for K in $2; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o gpurun_out/${TAG}_${K} -f python tools/profile_step.py --config $CFG > gpurun_out/${TAG}_${K}.log 2>&1
  echo "$K exit $?"
done
