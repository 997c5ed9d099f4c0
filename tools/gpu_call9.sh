#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python tools/step_series.py --config 3 --n 6 > gpurun_out/series9_c3_green.json 2>gpurun_out/series9_c3_green.err; cat gpurun_out/series9_c3_green.json; tail -2 gpurun_out/series9_c3_green.err
TN_NO_GREEN_CTX=1 timeout 300 python tools/step_series.py --config 3 --n 6 > gpurun_out/series9_c3_plain.json 2>gpurun_out/series9_c3_plain.err; cat gpurun_out/series9_c3_plain.json
timeout 300 python tools/step_series.py --config 2 --n 6 > gpurun_out/series9_c2_green.json 2>gpurun_out/series9_c2_green.err; cat gpurun_out/series9_c2_green.json
TN_NO_GREEN_CTX=1 timeout 300 python tools/step_series.py --config 2 --n 6 > gpurun_out/series9_c2_plain.json 2>gpurun_out/series9_c2_plain.err; cat gpurun_out/series9_c2_plain.json
timeout 300 python tools/env_time.py 3 haar > gpurun_out/env9_c3.json 2>&1; cat gpurun_out/env9_c3.json
TN_NO_GREEN_CTX=1 timeout 300 python tools/env_time.py 3 haar > gpurun_out/env9_c3_plain.json 2>&1; cat gpurun_out/env9_c3_plain.json
timeout 2400 python -m pytest tests -q -m gpu -rf --deselect "tests/test_gpu_full_parity.py::test_full_size_parity[c4]" --deselect "tests/test_gpu_full_parity.py::test_full_size_parity[c5r]" --deselect "tests/test_gpu_parity.py::test_full_size_properties_config5" > gpurun_out/gpu_tests_call9.log 2>&1; tail -6 gpurun_out/gpu_tests_call9.log
