# ncu --set full of the scan kernel at the bench config (llama) + summary; usage: bash scripts/ncu_scan.sh <tag>
T=${1:-x}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
  -o gpurun_out/${T}_scan_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/${T}_scan_full.log 2>&1; echo ncu scan rc=$?
python scripts/ncu_summary.py gpurun_out/${T}_scan_full.ncu-rep 25 > gpurun_out/${T}_scan_ncu_summary.txt 2>&1; head -32 gpurun_out/${T}_scan_ncu_summary.txt
