#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "low_entanglement or small-203 or small-202" > gpurun_out/sanitizer11.log 2>&1; echo "sanitizer rc=$?"; tail -8 gpurun_out/sanitizer11.log
timeout 900 python tools/tr_run.py --config 3 --problems 2 --outer 10 > gpurun_out/tr11_c3.json 2> gpurun_out/tr11_c3.err; python -c "
import json
d=json.loads(open('gpurun_out/tr11_c3.json').read().strip().splitlines()[-1])
print([(r['f0'],r['f'],r['hvps'],round(r['seconds'],1)) for r in d['rank0_runs']], d['wall_s'])"
timeout 900 python tools/tr_risk.py > gpurun_out/tr11_risk.json 2> gpurun_out/tr11_risk.err; tail -c 600 gpurun_out/tr11_risk.json
