python bench.py --steps 10 --warmup 3 > gpurun_out/r01x_bench.json 2> gpurun_out/r01x_bench.err; tail -c 2500 gpurun_out/r01x_bench.json
timeout 1200 python tools/config_report.py --out gpurun_out/r01x_configs.json 2>&1 | cut -c1-330
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01x_launches.csv python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_base_case -s 1 -c 1 -o gpurun_out/r01x_base2 -f python tools/profile_step.py --config 2 > /dev/null 2>&1; echo $?
