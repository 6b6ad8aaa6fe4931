timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 1 2 3 4 5; do python tools/profile_step.py --config $c 2>&1 | tail -1; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['base_ms_per_step'], d['e2e']['value'])"
