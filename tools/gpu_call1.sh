#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in 256 512 1024; do timeout 120 tools/eig_probe $n; done > gpurun_out/eig_probe.json 2>&1
cat gpurun_out/eig_probe.json
timeout 300 python tools/step_time.py --config 3 --reps 3 --tag prio > gpurun_out/st_c3_prio.json 2>gpurun_out/st_c3_prio.err; cat gpurun_out/st_c3_prio.json
TN_NO_STREAM_PRIO=1 timeout 300 python tools/step_time.py --config 3 --reps 3 --tag noprio > gpurun_out/st_c3_noprio.json 2>gpurun_out/st_c3_noprio.err; cat gpurun_out/st_c3_noprio.json
timeout 600 python tools/step_time.py --config 4 --reps 1 --tag prio > gpurun_out/st_c4_prio.json 2>gpurun_out/st_c4_prio.err; cat gpurun_out/st_c4_prio.json
TN_NO_STREAM_PRIO=1 timeout 600 python tools/step_time.py --config 4 --reps 1 --tag noprio > gpurun_out/st_c4_noprio.json 2>gpurun_out/st_c4_noprio.err; cat gpurun_out/st_c4_noprio.json
TN_PHASES=1 timeout 600 python tools/run_config.py --config 4 --max-batch 32 > gpurun_out/phases_c4.json 2> gpurun_out/phases_c4.err; cat gpurun_out/phases_c4.json; grep phases gpurun_out/phases_c4.err
timeout 2700 python -m pytest tests -q -m gpu -rf --deselect "tests/test_gpu_full_parity.py::test_full_size_parity[c4]" --durations=15 > gpurun_out/gpu_tests_call1.log 2>&1; tail -30 gpurun_out/gpu_tests_call1.log
