# round-2 GPU call 5: N4 (library TEBD) parity, N1 bench, C4 bench with the library-built reference
python -m paper_2604_20384_b200.build
python -m pytest tests/test_gpu_tebd.py tests/test_gpu_risk.py -x -q > gpurun_out/g5_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/g5_pytest.log
python bench.py --workload n1 --samples 8 --batch 4 --steps 1 --warmup 1 > gpurun_out/g5_bench_n1.json 2> gpurun_out/g5_bench_n1.err; echo n1_rc=$?
tail -c 1800 gpurun_out/g5_bench_n1.json; tail -3 gpurun_out/g5_bench_n1.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g5_bench_c4.json 2> gpurun_out/g5_bench_c4.err; echo c4_rc=$?
head -c 1200 gpurun_out/g5_bench_c4.json; tail -3 gpurun_out/g5_bench_c4.err
