# ncu --set full of the scan on the full config for variants: bash scripts/ab_ncu_full.sh <config> v1 v2 ...
mkdir -p gpurun_out
CFG=$1; shift
for v in "$@"; do
PASTA_LIB=build/variants/libpasta_$v.so timeout 1200 ncu --set full --import-source on --clock-control none -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/abf_${CFG}_$v python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo $v rc=$?
done
