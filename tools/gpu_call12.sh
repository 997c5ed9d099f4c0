#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_risk.py "tests/test_gpu_full_parity.py::test_full_size_parity[c3]" -q -m gpu -rf -x --deselect "tests/test_gpu_parity.py::test_full_size_properties_config5" > gpurun_out/gpu_tests_call12.log 2>&1; tail -5 gpurun_out/gpu_tests_call12.log
timeout 600 python tools/step_time.py --config 4 --reps 2 --ref tebd --tag gate2 > gpurun_out/st12_c4.json 2>gpurun_out/st12_c4.err; cat gpurun_out/st12_c4.json
