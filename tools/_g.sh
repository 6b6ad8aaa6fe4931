timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in default k512; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=$PWD/paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  echo "== $v"
  python tools/profile_step.py --config 2; python tools/profile_step.py --config 3; python tools/profile_step.py --config 5
  python tools/trace_levels.py 3 2> gpurun_out/r01i_trace3_$v.txt >/dev/null
done
unset DFGTB_LIB
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
