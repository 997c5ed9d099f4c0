#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py "tests/test_gpu_full_parity.py::test_full_size_parity[c3]" -q -m gpu -rf -x --durations=5 > gpurun_out/gpu_tests_call2.log 2>&1; tail -15 gpurun_out/gpu_tests_call2.log
timeout 300 python tools/step_time.py --config 2 --reps 3 --tag fast > gpurun_out/st2_c2_fast.json 2>gpurun_out/st2_c2_fast.err; cat gpurun_out/st2_c2_fast.json
TN_NO_CHOLQR=1 TN_NO_LOWDIN_LQ=1 timeout 300 python tools/step_time.py --config 2 --reps 3 --tag house > gpurun_out/st2_c2_house.json 2>gpurun_out/st2_c2_house.err; cat gpurun_out/st2_c2_house.json
timeout 300 python tools/step_time.py --config 3 --reps 3 --tag fast > gpurun_out/st2_c3_fast.json 2>gpurun_out/st2_c3_fast.err; cat gpurun_out/st2_c3_fast.json
TN_NO_CHOLQR=1 timeout 300 python tools/step_time.py --config 3 --reps 3 --tag nochol > gpurun_out/st2_c3_nochol.json 2>gpurun_out/st2_c3_nochol.err; cat gpurun_out/st2_c3_nochol.json
TN_NO_CHOLQR=1 TN_NO_LOWDIN_LQ=1 timeout 300 python tools/step_time.py --config 3 --reps 3 --tag house > gpurun_out/st2_c3_house.json 2>gpurun_out/st2_c3_house.err; cat gpurun_out/st2_c3_house.json
timeout 600 python tools/step_time.py --config 4 --reps 1 --tag fast > gpurun_out/st2_c4_fast.json 2>gpurun_out/st2_c4_fast.err; cat gpurun_out/st2_c4_fast.json
timeout 600 python tools/env_time.py 5 trotter > gpurun_out/env2_c5.json 2>&1; cat gpurun_out/env2_c5.json
