# compute-sanitizer runs over the small GPU parity tests (memcheck, racecheck, synccheck)
mkdir -p gpurun_out
K='hand_worked or snapshot or tiny_config or adversarial_random or contention or host_records or topk_direct or bitmap_or or topk_merge'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" -p no:cacheprovider > gpurun_out/san_$tool.log 2>&1
  echo $tool rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_$tool.log | tail -3
done
