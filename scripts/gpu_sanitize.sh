# compute-sanitizer runs over the small GPU parity tests (memcheck, racecheck, synccheck, initcheck)
mkdir -p gpurun_out
T=${1:-r02}
K='hand_worked or snapshot or tiny_config or adversarial_random or contention or host_records or topk_direct or topk_distributions or topk_unaligned or topk_many or bitmap_or or topk_merge or streaming'
KR='spec_range_filter or random_rich or tiny_rich'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" -p no:cacheprovider > gpurun_out/san_${T}_$tool.log 2>&1
  echo $tool parity rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${T}_$tool.log | tail -3
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_rich.py -m gpu -x -q -k "$KR" -p no:cacheprovider > gpurun_out/san_${T}_rich_$tool.log 2>&1
  echo $tool rich rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${T}_rich_$tool.log | tail -3
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_peer.py tests/test_gpu_report_usage.py -m gpu -x -q -k "sum_bitmap or world1 or streams or small_slots or gather" -p no:cacheprovider > gpurun_out/san_${T}_peer_$tool.log 2>&1
  echo $tool peer rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${T}_peer_$tool.log | tail -3
done
# the persistent streaming consumer (spin-waits on host-published descriptors): memcheck only
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stream_ring_equals and 4096-64" -p no:cacheprovider > gpurun_out/san_${T}_stream_memcheck.log 2>&1
echo memcheck stream rc=$?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${T}_stream_memcheck.log | tail -3
