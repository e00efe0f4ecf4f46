mkdir -p gpurun_out
./scripts/micro/red_rate | tee gpurun_out/red_rate.txt
PASTA_STREAM_DEFER_LAUNCH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 \
  -o gpurun_out/stream_full python scripts/stream_ring_bench.py 536870912 524288:1024 > gpurun_out/stream_ncu.log 2>&1; echo ncu rc=$?
python scripts/ncu_summary.py gpurun_out/stream_full.ncu-rep 40 > gpurun_out/stream_ncu_summary.txt 2>&1; head -30 gpurun_out/stream_ncu_summary.txt
