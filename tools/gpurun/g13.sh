# round-2 GPU call 13: C3 fused vs unfused step, pool reuse policy A/B
python -m paper_2604_20384_b200.build
for mode in "" "--unfused"; do for pool in 0 1; do
  if [ $pool = 1 ]; then export TN_POOL_STRICT=1; else unset TN_POOL_STRICT; fi
  python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $mode > gpurun_out/g13.json 2>/dev/null
  echo "mode=[$mode] strict_pool=$pool $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/g13.json)"
done; done
