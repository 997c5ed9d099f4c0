# round-2 GPU call 7: GEMM variant A/B (B-sum plane in shared memory) on hot shapes and a C4 apply
python -m paper_2604_20384_b200.build
python tools/gemm_bench.py > gpurun_out/g7_gemm_default.json; cat gpurun_out/g7_gemm_default.json
TN_GEMM_BSUM=1 python tools/gemm_bench.py > gpurun_out/g7_gemm_bsum.json; cat gpurun_out/g7_gemm_bsum.json
TN_GEMM_BSUM=1 python -m pytest tests/test_gpu_kernels.py -q -x -k zgemm 2>&1 | tail -2
python tools/ncu_apply.py --config 4 2>&1 | tail -1
TN_GEMM_BSUM=1 python tools/ncu_apply.py --config 4 2>&1 | tail -1
python -m pytest tests/test_gpu_tebd.py -q -x > gpurun_out/g7_tebd.log 2>&1; echo tebd_rc=$?; grep -E "^E |passed|failed" gpurun_out/g7_tebd.log | head -5
python bench.py --workload n1 --samples 4 --batch 4 --steps 1 --warmup 1 > gpurun_out/g7_bench_n1.json 2> gpurun_out/g7_bench_n1.err; echo n1_rc=$?
tail -c 1500 gpurun_out/g7_bench_n1.json; grep -v "^ " gpurun_out/g7_bench_n1.err | tail -3
