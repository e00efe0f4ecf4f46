for v in "$@"; do echo "== $v"; PASTA_LIB=build/variants/libpasta_$v.so timeout 600 python scripts/scan_sizes.py; done
