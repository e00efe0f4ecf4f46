mkdir -p gpurun_out
{ for a in "8388608 0" "8388608 1476618" "33554432 0" "1073741824 0"; do timeout 300 python scripts/warp_slow.py $a; done; } > gpurun_out/slow.log 2>&1
