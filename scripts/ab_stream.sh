# usage: bash scripts/ab_stream.sh v1 v2 ...   (A/B streaming mode: llama at 512 Ki-record batches)
for v in "$@"; do
  PASTA_LIB=build/variants/libpasta_$v.so timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --stream-batch 524288 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stream']; print('$v', 'step %.3f ms' % d['ms_per_step'], 'graph %.2f ms (%.2f us/call)' % (s['graph_ms'], s['graph_us_per_call']), 'eager %.2f ms' % s['eager_ms'])"
done
