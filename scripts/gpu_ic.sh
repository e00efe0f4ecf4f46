mkdir -p gpurun_out
{
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python scripts/rich_bench.py gpt2m
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['gpu_launches'])"
} > gpurun_out/ic.log 2>&1
