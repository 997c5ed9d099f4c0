# round-2 GPU call 1: suite on the refactored boundary, then ncu of the apply GEMM population at C4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2604_20384_b200.build
python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/g1_pytest.log
TN_GEMM_LOG=gpurun_out/apply_gemm_c4.log python tools/ncu_apply.py --config 4 > gpurun_out/g1_plain.log 2>&1 && \
TN_GEMM_LOG=gpurun_out/apply_gemm_c4_ncu.log ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:zgemm3m --launch-skip 6000 --launch-count 40 -o gpurun_out/zgemm_apply_c4 python tools/ncu_apply.py --config 4 > gpurun_out/g1_ncu.log 2>&1
echo ncu_rc=$?
tail -2 gpurun_out/g1_plain.log
