# round-2 GPU call 14: device-side frozen factors + point-free apply graphs: GPU suite, C2 / C3 / C4 bench
python -m paper_2604_20384_b200.build
python -m pytest tests -m gpu -x -q -k "not c4] and not c5r]" > gpurun_out/g14_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/g14_pytest.log; grep -E "^E |^FAILED" gpurun_out/g14_pytest.log | head -6
for c in 2 3; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g14_bench_c$c.json 2> gpurun_out/g14_bench_c$c.err; echo c${c}_rc=$?; grep -o '"ms_per_step": [0-9.]*' gpurun_out/g14_bench_c$c.json; grep -o '"phases": {[^}]*}' gpurun_out/g14_bench_c$c.json | cut -c1-200; tail -2 gpurun_out/g14_bench_c$c.err; done
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g14_bench_c4.json 2> gpurun_out/g14_bench_c4.err; echo c4_rc=$?; grep -o '"ms_per_step": [0-9.]*' gpurun_out/g14_bench_c4.json
