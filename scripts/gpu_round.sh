mkdir -p gpurun_out
set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm --format=csv
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config" > gpurun_out/pytest_small.log 2>&1; echo small rc=$?
tail -30 gpurun_out/pytest_small.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-sample 16777216 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
