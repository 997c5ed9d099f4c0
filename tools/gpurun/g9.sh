# round-2 GPU call 9: whole-step kernel shares at C4 (CUPTI) and the ncu launch list head of the bench command
python -m paper_2604_20384_b200.build
python tools/kprof.py --config 4 --what step --batch 64 --max-batch 32 > gpurun_out/g9_kprof_step_c4.txt 2>&1; echo kprof_rc=$?
head -30 gpurun_out/g9_kprof_step_c4.txt
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g9_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g9_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g9_ncu.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/g9_launches.csv
