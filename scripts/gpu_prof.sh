# usage: bash scripts/gpu_prof.sh <tag> [extra bench args]
mkdir -p gpurun_out
TAG=${1:-prof}
shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/${TAG}_scan python bench.py --n 1073741824 --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/${TAG}_prof.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/${TAG}_prof.log | cut -c1-300
