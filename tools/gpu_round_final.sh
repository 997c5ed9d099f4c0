#!/bin/bash
# End-of-round GPU batch: full GPU suite, smoke, environment timings, default bench + reference arm.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/gpu_tests_final.log 2>&1; tail -4 gpurun_out/gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -2
for c in 3 4; do timeout 300 python tools/env_time.py $c haar > gpurun_out/env_final_c$c.json 2>&1; cat gpurun_out/env_final_c$c.json; done
timeout 600 python tools/env_time.py 5 trotter > gpurun_out/env_final_c5.json 2>&1; cat gpurun_out/env_final_c5.json
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; cat gpurun_out/bench_final.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err; cat gpurun_out/bench_final_ref.json
