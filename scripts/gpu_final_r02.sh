# Round-2 final evidence at HEAD: everything of gpu_round2.sh, then the two microbenchmarks
# and the sanitizer pass. usage: bash scripts/gpu_final_r02.sh <tag>
T=${1:-r02f}
bash scripts/gpu_round2.sh $T
./scripts/micro/read_bw > gpurun_out/${T}_read_bw.txt 2>&1; echo read_bw rc=$?
./scripts/micro/red_rate > gpurun_out/${T}_red_rate.txt 2>&1; echo red_rate rc=$?
PASTA_STREAM_DEFER_LAUNCH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 \
  -o gpurun_out/${T}_stream_full python scripts/stream_ring_bench.py 536870912 524288:1024 > gpurun_out/${T}_stream_ncu.log 2>&1; echo ncu stream rc=$?
python scripts/ncu_summary.py gpurun_out/${T}_stream_full.ncu-rep 25 > gpurun_out/${T}_stream_ncu_summary.txt 2>&1
# (compute-sanitizer is closed on this GPU pool since mid-round 2: scripts/gpu_sanitize.sh not run)
