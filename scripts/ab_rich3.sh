for rep in 1 2; do
for v in "$@"; do
  lib=build/variants/libpasta_$v.so; [ "$v" = base ] && lib=paper_2602_22103_b200/libpasta.so
  for mb in "0 0" "0.05 0" "0.05 5"; do
    echo "$v $mb: $(PASTA_LIB=$lib timeout 300 python scripts/rich_bench.py gpt2m 2000000000 $mb 2>&1 | tail -1 | cut -c60-200)"
  done
done
done
