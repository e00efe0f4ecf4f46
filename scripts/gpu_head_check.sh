mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/h_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/h_pytest.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/h_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo bench rc=$?; tail -2 gpurun_out/h_bench.err
python -c "import json; d=json.load(open('gpurun_out/h_bench.json')); print(round(d['value'],1), d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'], d['cpu_baseline']['value'], d['e2e']['value'])"
