mkdir -p gpurun_out
for v in "$@"; do
PASTA_LIB=build/variants/libpasta_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk_$v.csv -k regex:'bitlen|digit|select|eq_count|gather|pad|bitonic|write|bitmap|footprint' python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo $v rc=$?
done
