for v in default sk0 sk2 sk3; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r03p_launches_$v.csv python tools/profile_step.py > /dev/null 2>&1
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['base_ms_per_step'], d['e2e']['value'])"
  python tools/profile_step.py --config 3 | tail -1; python tools/profile_step.py --config 5 | tail -1
done
