# usage: bash scripts/gpu_check.sh <tag> [pytest-k-expr]
mkdir -p gpurun_out
TAG=${1:-run}
K=${2:-}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/${TAG}_smoke.log
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
else
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
fi
tail -25 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-sample 16777216 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
