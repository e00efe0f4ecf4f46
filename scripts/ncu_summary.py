"""Summarise an ncu report: key metrics + SASS hot spots. usage: ncu_summary.py rep.ncu-rep [topn]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = det[0]; isec = h.index("Section Name"); iname = h.index("Metric Name"); iu = h.index("Metric Unit"); iv = h.index("Metric Value")
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
        "Achieved Active Warps Per SM", "L2 Hit Rate", "Avg. Active Threads Per Warp"]
for r in det[1:]:
    if len(r) > iv and r[iname] in want:
        print(f"{r[iname]:40s} {r[iv]:>16s} {r[iu]}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
if raw:
    hh = raw[0]; vals = raw[2] if len(raw) > 2 else raw[1]
    for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_requests_srcunit_tex_op_red.sum",
                "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum", "lts__t_requests_srcunit_tex_op_atom_dot_cas.sum",
                "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed",
                "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_requests_srcunit_tex_op_read.sum",
                "smsp__inst_executed.sum", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "smsp__average_warp_latency_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard"]:
        for i, name in enumerate(hh):
            if name == key:
                print(f"{key:55s} {vals[i]:>20s} {raw[1][i]}")
# stall reasons
for r in det[1:]:
    if len(r) > iv and r[isec] == "Warp State Statistics" and "Stall" in r[iname]:
        print(r[iname], r[iv])
sass = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
hdr = sass[1]; data = sass[2:]
ia = hdr.index("Address"); isrc = hdr.index("Source"); ist = hdr.index("Warp Stall Sampling (All Samples)"); iex = hdr.index("Instructions Executed")
tot_s = sum(float(r[ist] or 0) for r in data); tot_e = sum(float(r[iex] or 0) for r in data)
print("total stall samples", tot_s, "executed warp-instr", tot_e)
cur = None; out = []
for r in data:
    e = int(float(r[iex] or 0)); s = float(r[ist] or 0)
    if e != cur:
        if cur is not None: out.append(blk)
        cur = e; blk = [r[ia][-5:], 0, e, 0.0, r[isrc][:60]]
    blk[1] += 1; blk[3] += s
out.append(blk)
for b in sorted(out, key=lambda b: -(b[1] * b[2]))[:topn]:
    print(f"{b[0]} n={b[1]:3d} exec={b[2]:9d} instr%={100*b[1]*b[2]/tot_e:5.1f} stall%={100*b[3]/tot_s:5.1f} {b[4]}")
