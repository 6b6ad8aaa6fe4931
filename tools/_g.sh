timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_traverse -s 1 -c 1 -o gpurun_out/r01s_trav2 -f python tools/profile_step.py --config 2 > /dev/null 2>&1; echo $?
