# usage: bash scripts/ab.sh <config> v1 v2 ...   (A/B the scan variants under build/variants; base = the in-tree build)
mkdir -p gpurun_out
CFG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  lib=build/variants/libpasta_$v.so; [ "$v" = base ] && lib=paper_2602_22103_b200/libpasta.so
  r=$(PASTA_LIB=$lib timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu 2>>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms scan  %.1f GB/s  %.3f frac  step %.3f ms' % (d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['ms_per_step']))")
  echo "$CFG $v: $r"
done
done
