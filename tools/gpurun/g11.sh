# round-2 GPU call 11: split primal (two contexts), edge cases, whole GPU suite minus the pending goldens
python -m paper_2604_20384_b200.build
python -m pytest tests -m gpu -x -q -k "not c4] and not c5r]" > gpurun_out/g11_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/g11_pytest.log; grep -E "^E |^FAILED" gpurun_out/g11_pytest.log | head -6
