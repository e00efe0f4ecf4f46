# Copy one evidence run (gpurun_out/<tag>_*) into profiles/r02_* and regenerate the doc tables.
# usage: bash scripts/evidence_to_profiles.sh <tag>
T=$1; G=gpurun_out; P=profiles
cp $G/${T}_bench.json $P/r02_bench.json
for c in rn50 gpt2m uvm s_perm s_hot s_manyranges; do cp $G/${T}_cfg_$c.json $P/r02_configs/$c.json; done
cp $G/${T}_launches_summary.txt $P/r02_launches_summary.txt
cp $G/${T}_scan_ncu_summary.txt $P/r02_scan_ncu_summary.txt; cp $G/${T}_scan_full.ncu-rep $P/r02_scan_full.ncu-rep
cp $G/${T}_topk_ncu_summary.txt $P/r02_topk_ncu_summary.txt; cp $G/${T}_topk_full.ncu-rep $P/r02_topk_full.ncu-rep
cp $G/${T}_stream_ring.jsonl $P/r02_stream_ring.jsonl; cp $G/${T}_stream.json $P/r02_stream.json
cp $G/${T}_next.jsonl $P/r02_next_rows.jsonl; cp $G/${T}_reference.json $P/r02_reference.json
cp $G/${T}_read_bw.txt $P/r02_read_bw.txt; cp $G/${T}_red_rate.txt $P/r02_stress/red_rate.txt
cp $G/${T}_stream_ncu_summary.txt $P/r02_stream_ncu_summary.txt; cp $G/${T}_stream_full.ncu-rep $P/r02_stream_full.ncu-rep
cp $G/${T}_pytest.log $P/r02_gputest.log
python scripts/docs_tables.py $T
python - <<'PY'
import json, re
t = open('profiles/r02_scan_ncu_summary.txt').read()
rd = float(re.search(r'dram__bytes_read.sum\s+([\d.]+)\s+Gbyte', t).group(1))
wr = float(re.search(r'dram__bytes_write.sum\s+([\d.]+)\s+Mbyte', t).group(1))
tot = int(rd * 1e9 + wr * 1e6)
json.dump({'llama': tot, '_note': f'dram read + write bytes of one scan_kernel launch at the bench config (profiles/r02_scan_ncu_summary.txt: {rd} GB + {wr} MB); algorithmic 85,899,345,920 B (ratio {tot / 85899345920:.3f})'}, open('profiles/scan_traffic.json', 'w'), indent=1)
PY
