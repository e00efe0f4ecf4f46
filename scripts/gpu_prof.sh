mkdir -p gpurun_out
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_bench.json 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/prof_scan python bench.py --n 1073741824 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_scan.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/prof_scan.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "full_config" > gpurun_out/pytest_full.log 2>&1; echo full rc=$?
tail -15 gpurun_out/pytest_full.log
