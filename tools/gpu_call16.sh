#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python tools/env_time.py 5 trotter > gpurun_out/env16_c5.json 2>&1; cat gpurun_out/env16_c5.json
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py "tests/test_gpu_full_parity.py::test_full_size_parity[c3]" "tests/test_gpu_full_parity.py::test_full_size_parity[c5r]" -q -m gpu -rf -x --deselect "tests/test_gpu_parity.py::test_full_size_properties_config5" > gpurun_out/gpu_tests_call16.log 2>&1; tail -5 gpurun_out/gpu_tests_call16.log
