# Round evidence: tests, bench, launch list and a full ncu capture of the scan at the bench config.
# usage: bash scripts/gpu_evidence.sh <tag>
mkdir -p gpurun_out
TAG=${1:-ev}
bash scripts/gpu_check.sh "$TAG"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_launches_bench.json 2>&1; echo launches rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
  -o gpurun_out/${TAG}_scan_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${TAG}_scan_full.log 2>&1; echo ncu_full rc=$?
tail -2 gpurun_out/${TAG}_scan_full.log | cut -c1-200
