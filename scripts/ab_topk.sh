# usage: bash scripts/ab_topk.sh v1 v2 ...  (A/B top-K / finalize variants under build/variants; bench phases)
mkdir -p gpurun_out
for CFG in llama rn50 uvm gpt2m; do
for rep in 1 2; do
for v in "$@"; do
  lib=build/variants/libpasta_$v.so; [ "$v" = base ] && lib=paper_2602_22103_b200/libpasta.so
  r=$(PASTA_LIB=$lib timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('step %.4f  scan %.4f  finalize %.4f  topk %.4f  G rec/s %.1f' % (d['ms_per_step'], p['scan'], p['finalize'], p['topk'], d['value']))")
  echo "$CFG $v: $r"
done
done
done
