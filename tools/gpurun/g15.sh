# round-2 GPU call 15: ncu --set full over C3 apply GEMM launches (traffic_c3.json, same population as roofline.achieved)
python -m paper_2604_20384_b200.build
TN_GEMM_LOG=gpurun_out/apply_gemm_c3.log python tools/ncu_apply.py --config 3 > gpurun_out/g15_plain.log 2>&1 && \
TN_GEMM_LOG=gpurun_out/apply_gemm_c3_ncu.log ncu --profile-from-start off --set full --clock-control none \
  -k regex:zgemm3m --launch-skip 3000 --launch-count 16 -o /tmp/zgemm_apply_c3 python tools/ncu_apply.py --config 3 > gpurun_out/g15_ncu.log 2>&1
echo ncu_rc=$?
ncu -i /tmp/zgemm_apply_c3.ncu-rep --page raw --csv > gpurun_out/zgemm_apply_c3_raw.csv 2>&1
tail -1 gpurun_out/g15_plain.log; wc -l gpurun_out/apply_gemm_c3_ncu.log
