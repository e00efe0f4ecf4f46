# usage: bash scripts/ab_rich.sh v1 v2 ...   (A/B rich-scan variants under build/variants, twice each)
for rep in 1 2; do
for v in "$@"; do
  echo "== $v"
  PASTA_LIB=build/variants/libpasta_$v.so timeout 300 python scripts/next_bench.py --only rich 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print(d['variant'], d['scan_ms'], d['frac'])
    except Exception:
        print(l.strip())
"
done
done
