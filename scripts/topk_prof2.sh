mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/topk_coop.csv -k regex:'select_coop|pad|bitonic|write|bitmap|footprint' python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'select_coop' -s 1 -c 1 -o gpurun_out/topk_coop python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo rc=$?
