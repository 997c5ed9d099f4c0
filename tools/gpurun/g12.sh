# round-2 GPU call 12: C2 / C3 bench lines, N1 with 4 samples in flight
python -m paper_2604_20384_b200.build
for c in 2 3; do python bench.py --config $c --steps 2 --warmup 3 > gpurun_out/g12_bench_c$c.json 2> gpurun_out/g12_bench_c$c.err; echo c${c}_rc=$?; head -c 300 gpurun_out/g12_bench_c$c.json; echo; grep -o '"phases": {[^}]*}' gpurun_out/g12_bench_c$c.json; grep -o '"step_frac": [0-9.]*' gpurun_out/g12_bench_c$c.json; grep -o '"frac": [0-9.]*' gpurun_out/g12_bench_c$c.json; done
python bench.py --workload n1 --samples 4 --batch 4 --concurrency 4 --steps 1 --warmup 1 > gpurun_out/g12_bench_n1_c4.json 2> gpurun_out/g12_bench_n1.err; echo n1_rc=$?
head -c 400 gpurun_out/g12_bench_n1_c4.json; grep -o '"phases": {[^}]*}' gpurun_out/g12_bench_n1_c4.json; tail -2 gpurun_out/g12_bench_n1.err
