# round-2 GPU call 3: regression of the site-dim refactor (whole GPU suite), full-size C3 parity, primal timelines
python -m paper_2604_20384_b200.build
python -m pytest tests -m gpu -x -q -k "not full_size_parity" > gpurun_out/g3_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/g3_pytest.log
python -m pytest tests/test_gpu_full_parity.py -k c3 -x -q -s > gpurun_out/g3_fullparity_c3.log 2>&1; echo fullparity_rc=$?
grep -E "case|passed|failed|Error" gpurun_out/g3_fullparity_c3.log | head -5
python tools/timeline.py --config 4 --what env > gpurun_out/g3_timeline_c4_env.json 2> gpurun_out/g3_timeline.err; echo tl_rc=$?
python tools/timeline.py --config 3 --what step > gpurun_out/g3_timeline_c3_step.json 2>> gpurun_out/g3_timeline.err
head -c 1500 gpurun_out/g3_timeline_c4_env.json
