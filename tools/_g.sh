timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\.\|passed" | tail -30
python -c "
import sys; sys.path.insert(0,'.')
from paper_1102_2878_b200 import _capi; print('mufu err', _capi.lib.dfgtb_mufu_exp_error())"
for c in 2 3 4 5; do python tools/profile_step.py --config $c; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'], d['e2e']['value'], d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_base_case -s 1 -c 1 -o gpurun_out/r01q_base2 -f python tools/profile_step.py --config 2 > /dev/null 2>&1; echo $?
