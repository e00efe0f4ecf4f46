# tests + profile: usage bash scripts/gpu_tp.sh <tag>
mkdir -p gpurun_out
TAG=$1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?; tail -14 gpurun_out/${TAG}_pytest.log
bash scripts/gpu_prof.sh $TAG
