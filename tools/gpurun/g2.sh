# round-2 GPU call 2: new tests (ABI, full-size C3 parity), CPU reference build time on the box, bench C3, ncu apply sample
nproc; grep -m1 "model name" /proc/cpuinfo
python -m paper_2604_20384_b200.build
python -m pytest tests/test_gpu_full_parity.py -k c3 -x -q -s > gpurun_out/g2_fullparity_c3.log 2>&1; echo fullparity_rc=$?
tail -5 gpurun_out/g2_fullparity_c3.log
python -m pytest tests/test_gpu_abi.py tests/test_gpu_parity.py -x -q > gpurun_out/g2_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/g2_pytest.log
python -c "
import time,sys; sys.path.insert(0,'.')
from tn_inputs import configs as C
for cid in (4,5):
    t=time.time(); C.reference_mpo(C.CONFIGS[cid], device='cpu'); print('cpu reference build', cid, time.time()-t, flush=True)
" > gpurun_out/g2_refbuild.log 2>&1; cat gpurun_out/g2_refbuild.log
python bench.py --config 3 --steps 1 --warmup 3 > gpurun_out/g2_bench_c3.json 2> gpurun_out/g2_bench_c3.err; echo bench_rc=$?
tail -c 3000 gpurun_out/g2_bench_c3.json
python tools/ncu_apply.py --config 4 > gpurun_out/g2_plain.log 2>&1 && \
TN_GEMM_LOG=gpurun_out/apply_gemm_c4_ncu.log ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:zgemm3m --launch-skip 6000 --launch-count 12 -o /tmp/zgemm_apply_c4 python tools/ncu_apply.py --config 4 > gpurun_out/g2_ncu.log 2>&1
echo ncu_rc=$?
ncu -i /tmp/zgemm_apply_c4.ncu-rep --page raw --csv > gpurun_out/zgemm_apply_c4_raw.csv 2>&1
ncu -i /tmp/zgemm_apply_c4.ncu-rep --page details --csv > gpurun_out/zgemm_apply_c4_details.csv 2>&1
ls -la /tmp/zgemm_apply_c4.ncu-rep; cp /tmp/zgemm_apply_c4.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
