# usage: bash scripts/ab.sh <config> v1 v2 ...   (A/B the scan variants under build/variants)
mkdir -p gpurun_out
CFG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  r=$(PASTA_LIB=build/variants/libpasta_$v.so timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms scan  %.1f GB/s  %.3f frac  step %.3f ms' % (d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['ms_per_step']))")
  echo "$CFG $v: $r"
done
done
