#!/bin/bash
# Round-end evidence: GPU tests, the bench line, launch lists of cfg2 / cfg3 / cfg5, ncu
# --set full captures of the hot kernels (cfg2: base case, traversal; cfg3: expansion
# kernels and the FP32 base case), each only after its own command ran clean.
#   tools/gpu_profiles.sh TAG
TAG=${1:-r2d}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" | tee -a gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?"
for C in 2 3 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_cfg$C.csv python tools/profile_step.py --config $C > gpurun_out/${TAG}_launch_cfg$C.log 2>&1
  echo "launch list cfg$C exit $?"
done
cap() {  # cap NAME REGEX SKIP CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 \
    -o gpurun_out/${TAG}_$1 -f python tools/profile_step.py --config $4 > gpurun_out/${TAG}_$1.log 2>&1
  echo "ncu $1 exit $?"
  # summaries on the box (the reports themselves can exceed gpurun's 64 MiB return limit)
  python tools/ncu_summary.py gpurun_out/${TAG}_$1.ncu-rep > gpurun_out/${TAG}_$1_ncu.txt 2>&1
  ncu -i gpurun_out/${TAG}_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_sass.csv 2>/dev/null
  python tools/sass_blocks.py gpurun_out/${TAG}_$1_sass.csv 20 > gpurun_out/${TAG}_$1_sass_blocks.txt 2>&1
  rm -f gpurun_out/${TAG}_$1_sass.csv
  [ "$KEEP_REPS" = "1" ] || rm -f gpurun_out/${TAG}_$1.ncu-rep
}
cap cfg2_base_f32 "k_base_f32" 1 2
cap cfg2_base_case "k_base_case$" 1 2
cap cfg2_traverse "k_traverse" 1 2
cap cfg2_farfield "k_farfield_t" 1 2
cap cfg3_base_f32 "k_base_f32" 4 3
cap cfg3_farfield "k_farfield_t" 4 3
cap cfg3_local_chunks "k_local_chunks_w" 4 3
cap cfg3_finalize "k_finalize_t" 4 3
