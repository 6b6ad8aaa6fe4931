python -m pytest tests/test_gpu_f32.py tests/test_gpu_engine.py tests/test_gpu_fuzz.py tests/test_gpu_cv.py -x -q 2>&1 | tail -3
for v in default sb4; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['base_ms_per_step'], d['e2e']['value'])"
done
unset DFGTB_LIB
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03f_launches.csv python tools/profile_step.py > /dev/null 2>&1
python tools/phase_report.py --config 2 > gpurun_out/r03f_phase2.txt 2>&1
