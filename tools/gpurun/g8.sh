# round-2 GPU call 8: suite after the GEMM revert and TEBD tolerances; C4 sub-batch 64 experiment
python -m paper_2604_20384_b200.build
python -m pytest tests -m gpu -x -q -k "not c4] and not c5r]" > gpurun_out/g8_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/g8_pytest.log; grep -E "^E " gpurun_out/g8_pytest.log | head -3
python bench.py --steps 1 --warmup 2 --max-batch 64 --no-e2e --no-cpu-baseline > gpurun_out/g8_bench_c4_mb64.json 2> gpurun_out/g8_bench_c4_mb64.err; echo mb64_rc=$?
head -c 400 gpurun_out/g8_bench_c4_mb64.json; grep -o '"phases": {[^}]*}' gpurun_out/g8_bench_c4_mb64.json; tail -2 gpurun_out/g8_bench_c4_mb64.err
