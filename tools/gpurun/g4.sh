# round-2 GPU call 4: N1 state-mode parity, N1 bench line, C4 bench line with the new fields
python -m paper_2604_20384_b200.build
python -m pytest tests/test_gpu_risk.py tests/test_gpu_abi.py -x -q > gpurun_out/g4_pytest.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/g4_pytest.log
python bench.py --workload n1 --samples 8 --batch 8 --steps 1 --warmup 1 > gpurun_out/g4_bench_n1.json 2> gpurun_out/g4_bench_n1.err; echo n1_rc=$?
tail -c 1500 gpurun_out/g4_bench_n1.json; tail -5 gpurun_out/g4_bench_n1.err
python bench.py --steps 1 --warmup 3 > gpurun_out/g4_bench_c4.json 2> gpurun_out/g4_bench_c4.err; echo c4_rc=$?
head -c 800 gpurun_out/g4_bench_c4.json; tail -3 gpurun_out/g4_bench_c4.err
