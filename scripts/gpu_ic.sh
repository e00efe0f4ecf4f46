mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in llama uvm gpt2m rn50; do bash scripts/ab.sh $c c il nil; done
bash scripts/scan_sizes_ab.sh "llama 1048576 8388608 33554432" c il
} > gpurun_out/ic.log 2>&1
