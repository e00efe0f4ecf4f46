# Round evidence at HEAD: smoke, every GPU test, the bench line, NEXT-row measurements,
# the launch list and full ncu captures of the scan and rich kernels.
# usage: bash scripts/gpu_final.sh <tag>
mkdir -p gpurun_out
TAG=${1:-final}
bash scripts/gpu_evidence.sh "$TAG"
timeout 900 python scripts/next_bench.py > gpurun_out/${TAG}_next.jsonl 2> gpurun_out/${TAG}_next.err; echo next rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:rich_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_rich_full python scripts/rich_bench.py gpt2m 1000000000 0 0 > gpurun_out/${TAG}_rich_ncu.log 2>&1
echo rich ncu rc=$?
