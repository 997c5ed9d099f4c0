#!/bin/bash
# One gpurun batch: full GPU test suite, environment timing, fused vs unfused bench at C4, NEXT-row timings.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/gpu_tests_a.log 2>&1; tail -6 gpurun_out/gpu_tests_a.log
timeout 300 python tools/env_time.py 4 haar > gpurun_out/env_c4e.json 2>&1; cat gpurun_out/env_c4e.json
timeout 200 python tools/env_time.py 3 haar > gpurun_out/env_c3e.json 2>&1; cat gpurun_out/env_c3e.json
timeout 600 python bench.py > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err; cat gpurun_out/bench_c4_fused.json
timeout 600 python bench.py --unfused --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_unfused.json 2> gpurun_out/bench_c4_unfused.err; cat gpurun_out/bench_c4_unfused.json
timeout 400 python tools/next_rows_bench.py > gpurun_out/next_rows.json 2> gpurun_out/next_rows.err; cat gpurun_out/next_rows.json; tail -3 gpurun_out/next_rows.err
