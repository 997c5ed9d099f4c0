# round-2 GPU call 6: whole GPU suite (GEMM variant cleanup, pool reuse policy), N1 bench, C4 bench
python -m paper_2604_20384_b200.build
python -m pytest tests -m gpu -x -q -k "not c4] and not c5r]" > gpurun_out/g6_pytest.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/g6_pytest.log
python bench.py --workload n1 --samples 8 --batch 4 --steps 1 --warmup 1 > gpurun_out/g6_bench_n1.json 2> gpurun_out/g6_bench_n1.err; echo n1_rc=$?
tail -c 1500 gpurun_out/g6_bench_n1.json; tail -2 gpurun_out/g6_bench_n1.err
python bench.py --steps 1 --warmup 3 > gpurun_out/g6_bench_c4.json 2> gpurun_out/g6_bench_c4.err; echo c4_rc=$?
head -c 600 gpurun_out/g6_bench_c4.json; tail -2 gpurun_out/g6_bench_c4.err
