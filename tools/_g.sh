for v in default gm16m3 gm16m4; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=$PWD/paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  echo "== $v"; python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['base_ms_per_step'])"
done
