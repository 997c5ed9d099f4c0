#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/step_time.py --config 3 --reps 3 --ref tebd --tag tebd > gpurun_out/st6_c3_tebd.json 2>gpurun_out/st6_c3_tebd.err; cat gpurun_out/st6_c3_tebd.json
timeout 300 python tools/step_time.py --config 3 --reps 3 --ref torch --tag torch > gpurun_out/st6_c3_torch.json 2>gpurun_out/st6_c3_torch.err; cat gpurun_out/st6_c3_torch.json
TN_NO_LOWRANK=1 timeout 300 python tools/step_time.py --config 3 --reps 3 --ref tebd --tag tebd_nolowrank > gpurun_out/st6_c3_tebd_nl.json 2>gpurun_out/st6_c3_tebd_nl.err; cat gpurun_out/st6_c3_tebd_nl.json
timeout 600 python bench.py --config 3 --steps 3 --no-cpu-baseline > gpurun_out/bench6_c3.json 2> gpurun_out/bench6_c3.err; cat gpurun_out/bench6_c3.json
timeout 600 python tools/step_time.py --config 4 --reps 1 --ref tebd --tag tebd > gpurun_out/st6_c4_tebd.json 2>gpurun_out/st6_c4_tebd.err; cat gpurun_out/st6_c4_tebd.json
