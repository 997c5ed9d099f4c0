#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:"apply_gate" --launch-skip 2500 --launch-count 12 --csv --page raw --log-file gpurun_out/ncu_gate_c4.csv python tools/ncu_apply.py --config 4 --batch 32 > gpurun_out/ncu_gate_c4.log 2>&1; tail -2 gpurun_out/ncu_gate_c4.log
python tools/ncu_hbm_summary.py gpurun_out/ncu_gate_c4.csv > gpurun_out/ncu_gate_c4.md 2>&1; cat gpurun_out/ncu_gate_c4.md | cut -c1-200
