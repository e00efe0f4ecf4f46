# usage: bash scripts/ab_topk.sh v1 v2 ...   (A/B top-K variants under build/variants: llama step, top-K phase)
for rep in 1 2; do
for v in "$@"; do
  r=$(PASTA_LIB=build/variants/libpasta_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step %.3f ms  topk %.4f ms  finalize %.4f ms' % (d['ms_per_step'], d['phases_ms_per_step']['topk'], d['phases_ms_per_step']['finalize']))")
  echo "$v: $r"
done
done
