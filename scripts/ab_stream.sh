# usage: bash scripts/ab_stream.sh v1 v2 ...  (streaming ring consumer A/B; base = the in-tree build)
for rep in 1 2; do
for v in "$@"; do
  lib=build/variants/libpasta_$v.so; [ "$v" = base ] && lib=paper_2602_22103_b200/libpasta.so
  echo "$v: $(PASTA_LIB=$lib timeout 300 python scripts/stream_ring_bench.py 2147483648 524288:256 4194304:64 2>&1 | tail -2 | tr '\n' ' ')"
done
done
