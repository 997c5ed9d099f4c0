#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python tools/step_series.py --config 3 --n 10 > gpurun_out/series_c3.json 2>gpurun_out/series_c3.err; cat gpurun_out/series_c3.json
TN_NO_CHAIN_CACHE=1 timeout 300 python tools/step_series.py --config 3 --n 10 > gpurun_out/series_c3_nocache.json 2>gpurun_out/series_c3_nocache.err; cat gpurun_out/series_c3_nocache.json
timeout 600 python tools/step_series.py --config 4 --n 4 > gpurun_out/series_c4.json 2>gpurun_out/series_c4.err; cat gpurun_out/series_c4.json
