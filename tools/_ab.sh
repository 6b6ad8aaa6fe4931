for v in default minb5 minb6 f32m8 default minb5 minb6 f32m8; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); pk=d['roofline']['per_kernel']; print('$v', round(d['ms_per_step'],4), round(d['roofline']['base_ms_per_step'],4), [round(k['ms_per_step'],4) for k in pk], [round(k['frac'],3) for k in pk])"
done
