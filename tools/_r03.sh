bash tools/gpu_round.sh r03v > gpurun_out/r03v_round.log 2>&1
for c in 2 3 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r03v_kernels_cfg$c.csv python tools/profile_step.py --config $c > /dev/null 2>&1
done
for c in 1 2 3 4 5; do python tools/base_split.py --config $c | tail -1; done > gpurun_out/r03v_split.txt 2>&1
python tools/config_report.py > gpurun_out/r03v_configs.json 2> gpurun_out/r03v_configs.err
python tools/e2e_breakdown.py 2 > gpurun_out/r03v_e2e.txt 2>&1
