mkdir -p gpurun_out
{
for c in llama uvm gpt2m rn50; do bash scripts/ab.sh $c c i6 i7 i8 i9 i8c4; done
} > gpurun_out/ic.log 2>&1
