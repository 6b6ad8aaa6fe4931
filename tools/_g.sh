python bench.py --steps 10 --warmup 3 > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; tail -c 1800 gpurun_out/r02i_bench.json | head -c 900; echo
timeout 1200 python tools/config_report.py --out gpurun_out/r02i_configs.json 2>&1 | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launches.csv python tools/profile_step.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_base_case -s 1 -c 1 -o gpurun_out/r02i_base2 -f python tools/profile_step.py --config 2 > /dev/null 2>&1; echo $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 1 -c 1 -o gpurun_out/r02i_trav2 -f python tools/profile_step.py --config 2 > /dev/null 2>&1; echo $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_base_case -s 1 -c 1 -o gpurun_out/r02i_base3 -f python tools/profile_step.py --config 3 > /dev/null 2>&1; echo $?
