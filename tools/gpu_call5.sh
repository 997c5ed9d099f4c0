#!/bin/bash
# Round-2 final batch: full GPU suite, smoke, bench lines (C4 default + reference arm, C3, C2, N1), CUPTI shares, ncu launch window.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf --deselect "tests/test_gpu_full_parity.py::test_full_size_parity[c4]" --durations=8 > gpurun_out/gpu_tests_call5.log 2>&1; tail -14 gpurun_out/gpu_tests_call5.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench5_c4.json 2> gpurun_out/bench5_c4.err; cat gpurun_out/bench5_c4.json
timeout 900 python bench.py --impl reference > gpurun_out/bench5_c4_ref.json 2> gpurun_out/bench5_c4_ref.err; cat gpurun_out/bench5_c4_ref.json
timeout 600 python bench.py --config 3 --steps 3 > gpurun_out/bench5_c3.json 2> gpurun_out/bench5_c3.err; cat gpurun_out/bench5_c3.json
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/bench5_c2.json 2> gpurun_out/bench5_c2.err; cat gpurun_out/bench5_c2.json
timeout 900 python bench.py --workload n1 --samples 4 --batch 4 --no-cpu-baseline > gpurun_out/bench5_n1.json 2> gpurun_out/bench5_n1.err; cat gpurun_out/bench5_n1.json
timeout 600 python tools/kprof.py --config 4 --what step --batch 64 --max-batch 32 > gpurun_out/kprof5_step_c4.txt 2>&1; head -30 gpurun_out/kprof5_step_c4.txt
timeout 300 python tools/env_time.py 3 haar > gpurun_out/env5_c3.json 2>&1; cat gpurun_out/env5_c3.json
timeout 300 python tools/env_time.py 4 haar > gpurun_out/env5_c4.json 2>&1; cat gpurun_out/env5_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300000 -c 40000 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu5.log 2>&1; python tools/ncu_summary.py gpurun_out/launches5.csv > gpurun_out/launches5.md 2>&1; head -20 gpurun_out/launches5.md
