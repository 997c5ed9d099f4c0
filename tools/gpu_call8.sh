#!/bin/bash
cd "$(dirname "$0")/.."
for sms in 72 48 32; do timeout 60 tools/green_probe 1024 $sms; echo " rc=$?"; done > gpurun_out/green_probe.json 2>&1
timeout 60 tools/green_probe 512 72 >> gpurun_out/green_probe.json 2>&1; echo " rc=$?" >> gpurun_out/green_probe.json
cat gpurun_out/green_probe.json
nvidia-smi --query-gpu=name,memory.used --format=csv
