#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TN_SPLIT_LOG=gpurun_out/split_log_c5.txt timeout 600 python tools/env_time.py 5 trotter > gpurun_out/env4_c5.json 2>&1; cat gpurun_out/env4_c5.json
TN_DEFLATE_STEP=1e-6 timeout 600 python tools/env_time.py 5 trotter > gpurun_out/env4_c5_step6.json 2>&1; cat gpurun_out/env4_c5_step6.json
TN_DEFLATE_STEP=1e-6 timeout 900 python -m pytest "tests/test_gpu_full_parity.py::test_full_size_parity[c5r]" "tests/test_gpu_full_parity.py::test_full_size_parity[c3]" tests/test_gpu_parity.py -q -m gpu -rf -s -x > gpurun_out/gpu_tests_call4.log 2>&1; tail -5 gpurun_out/gpu_tests_call4.log | cut -c1-1500
