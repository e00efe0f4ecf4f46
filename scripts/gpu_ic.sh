mkdir -p gpurun_out
{
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for a in "0 0" "0.05 0" "0.05 5"; do timeout 600 python scripts/rich_bench.py gpt2m 0 $a; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['gpu_launches'])"
} > gpurun_out/ic.log 2>&1
