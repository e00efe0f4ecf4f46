# bench line of every BASELINE config (1 GPU): usage bash scripts/gpu_configs.sh <tag>
mkdir -p gpurun_out
for c in rn50 gpt2m uvm llama; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/${1}_cfg_$c.json 2> gpurun_out/${1}_cfg_$c.err; echo $c rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${1}_reference.json 2>&1; echo ref rc=$?
