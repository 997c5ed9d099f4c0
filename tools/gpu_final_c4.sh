#!/bin/bash
# C4 stored-oracle parity alone (quick feedback once tests/golden/full_c4*.npz exist)
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest "tests/test_gpu_full_parity.py::test_full_size_parity[c4]" -q -m gpu -rs -rf -s > gpurun_out/gpu_c4_parity.log 2>&1; tail -8 gpurun_out/gpu_c4_parity.log | cut -c1-2500
