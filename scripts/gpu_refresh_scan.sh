# Re-measure what a scan change moves: smoke, the bench line, every config / stress row,
# the launch list, ncu of the scan, NEXT rows. usage: bash scripts/gpu_refresh_scan.sh <tag>
T=${1:-r02g}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?; tail -2 gpurun_out/${T}_bench.err
python -c "import json; d=json.load(open('gpurun_out/${T}_bench.json')); print(round(d['value'],1), d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'], d['cpu_baseline']['value'], d['e2e']['value'])"
for c in rn50 gpt2m uvm s_perm s_hot s_manyranges; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_cfg_$c.json 2> gpurun_out/${T}_cfg_$c.err
  python -c "import json; d=json.load(open('gpurun_out/${T}_cfg_$c.json')); r=d['roofline']; print('$c', round(d['value'],1), round(d['ms_per_step'],4), 'scan', round(r['avg_launch_ms'],4), 'frac', round(r['frac'],3), {k: round(v,4) for k,v in d['phases_ms_per_step'].items() if v})"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${T}_launches_bench.json 2>&1; echo launches rc=$?
python scripts/launch_summary.py gpurun_out/${T}_launches.csv "python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu" > gpurun_out/${T}_launches_summary.txt; head -14 gpurun_out/${T}_launches_summary.txt
bash scripts/ncu_scan.sh $T
timeout 1200 python scripts/next_bench.py > gpurun_out/${T}_next.jsonl 2> gpurun_out/${T}_next.err; echo next rc=$?; cat gpurun_out/${T}_next.jsonl | cut -c1-200
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --stream-batch 524288 > gpurun_out/${T}_stream.json 2> gpurun_out/${T}_stream.err; echo stream rc=$?
