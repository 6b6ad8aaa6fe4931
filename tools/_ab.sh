for v in default t512x2 t256x4 t512x1 default t512x2; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['base_ms_per_step'],4), d['e2e']['value'], d['scores'][2]['lk'])"
  python tools/phase_report.py --config 3 2>/dev/null | python tools/show_phases.py /dev/stdin | tail -1
done
