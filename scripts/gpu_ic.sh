mkdir -p gpurun_out
{
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in llama uvm; do bash scripts/ab.sh $c il cur; done
} > gpurun_out/ic.log 2>&1
