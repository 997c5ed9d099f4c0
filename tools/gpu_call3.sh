#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_abi.py "tests/test_gpu_full_parity.py::test_full_size_parity[c3]" "tests/test_gpu_full_parity.py::test_full_size_parity[c5r]" -q -m gpu -rf -s --durations=5 > gpurun_out/gpu_tests_call3.log 2>&1; tail -15 gpurun_out/gpu_tests_call3.log; grep split_stats gpurun_out/gpu_tests_call3.log | cut -c1-600
timeout 600 python tools/env_time.py 5 trotter > gpurun_out/env3_c5.json 2>&1; cat gpurun_out/env3_c5.json
timeout 300 python tools/step_time.py --config 3 --reps 3 --tag lowrank > gpurun_out/st3_c3.json 2>gpurun_out/st3_c3.err; cat gpurun_out/st3_c3.json
timeout 600 python tools/step_time.py --config 4 --reps 1 --tag lowrank > gpurun_out/st3_c4.json 2>gpurun_out/st3_c4.err; cat gpurun_out/st3_c4.json
