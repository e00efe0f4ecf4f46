# ncu --set full of the scan for variants: bash scripts/ab_ncu.sh <config> v1 v2 ...
mkdir -p gpurun_out
CFG=$1; shift
for v in "$@"; do
PASTA_LIB=build/variants/libpasta_$v.so timeout 900 ncu --set full --clock-control none -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/ab_${CFG}_$v python bench.py --config $CFG --n 1073741824 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo $v rc=$?
done
