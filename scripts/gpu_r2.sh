mkdir -p gpurun_out
bash scripts/gpu_check.sh w24
for c in rn50 gpt2m uvm; do bash scripts/ab.sh $c w16 w24 w28 2>&1 | head -3; done
bash scripts/ab.sh llama w28 | head -1
