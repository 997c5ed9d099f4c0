#!/bin/bash
# End of round 2: the driver's sequence -- full GPU suite, smoke, default bench, reference arm.
cd "$(dirname "$0")/.."
timeout 3000 python -m pytest tests -x -q -m gpu -rs --durations=6 > gpurun_out/gpu_tests_last.log 2>&1; tail -14 gpurun_out/gpu_tests_last.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_last_c4.json 2> gpurun_out/bench_last_c4.err; cat gpurun_out/bench_last_c4.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_last_c4_ref.json 2> gpurun_out/bench_last_c4_ref.err; cat gpurun_out/bench_last_c4_ref.json
timeout 600 python bench.py --config 3 --steps 5 --no-cpu-baseline > gpurun_out/bench_last_c3.json 2> gpurun_out/bench_last_c3.err; cat gpurun_out/bench_last_c3.json | cut -c1-400
timeout 600 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/bench_last_c2.json 2> gpurun_out/bench_last_c2.err; cat gpurun_out/bench_last_c2.json | cut -c1-400
timeout 900 python bench.py --workload n1 --samples 4 --batch 4 --no-cpu-baseline > gpurun_out/bench_last_n1.json 2> gpurun_out/bench_last_n1.err; cat gpurun_out/bench_last_n1.json | cut -c1-400
