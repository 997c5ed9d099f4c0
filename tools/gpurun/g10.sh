# round-2 GPU call 10: two C3 trust-region problems concurrently on one B200 (vs 99 s each sequentially in round 1)
python -m paper_2604_20384_b200.build
python tools/tr_run.py --config 3 --problems 2 --outer 10 --concurrent 2 > gpurun_out/g10_tr_c3_conc2.json 2> gpurun_out/g10_tr.err; echo tr_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/g10_tr_c3_conc2.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('config','problems','concurrent','final_f','wall_s')}, [(r['problem'], r['hvps'], round(r['seconds'],1)) for r in d['rank0_runs']])"
tail -3 gpurun_out/g10_tr.err
