# round-2 GPU call 16: risk tests (incl. TR on the risk), the N1 training experiment at C3 width
python -m paper_2604_20384_b200.build
python -m pytest tests/test_gpu_risk.py -x -q > gpurun_out/g16_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/g16_pytest.log; grep -E "^E " gpurun_out/g16_pytest.log | head -5
timeout 1500 python tools/tr_risk.py --config 3 --train 8 --test 8 --outer 10 > gpurun_out/g16_tr_risk_c3.json 2> gpurun_out/g16_tr_risk.err; echo tr_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/g16_tr_risk_c3.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('config','train_risk','test_risk_start','test_risk_end','hvps','tr_seconds','wall_s')})"
tail -3 gpurun_out/g16_tr_risk.err
