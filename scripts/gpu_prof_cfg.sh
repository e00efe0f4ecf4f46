# ncu --set full of one scan launch for a config: bash scripts/gpu_prof_cfg.sh <tag> <config>
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/$1_$2 python bench.py --config $2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/$1_$2.log 2>&1; echo ncu rc=$?
