# Stress rows + per-config scan captures: full-size parity of the
# stress plans, one bench line each, and an ncu --set full capture of the scan per config.
# usage: bash scripts/gpu_stress.sh <tag> [configs]
mkdir -p gpurun_out
TAG=${1:-stress}
CFGS=${2:-"s_perm s_hot s_manyranges rn50 gpt2m uvm"}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_config_bit_exact and s_" \
  > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/${TAG}_pytest.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_${c}.json 2> gpurun_out/${TAG}_${c}.err
  echo "bench $c rc=$?"; python -c "import json,sys; d=json.load(open('gpurun_out/${TAG}_${c}.json')); r=d['roofline']; print('$c', round(d['value'],1), 'G rec/s', 'scan', round(r['avg_launch_ms'],3), 'ms', 'frac', round(r['frac'],3), d['phases_ms_per_step'])" 2>&1 | tail -1
done
for c in $CFGS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG}_${c}_scan python bench.py --config $c --steps 1 --warmup 1 --no-cpu --no-e2e \
    > gpurun_out/${TAG}_${c}_ncu.log 2>&1; echo "ncu $c rc=$?"
  python scripts/ncu_summary.py gpurun_out/${TAG}_${c}_scan.ncu-rep 12 > gpurun_out/${TAG}_${c}_scan_summary.txt 2>&1
done
