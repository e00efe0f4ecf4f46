"""Per-basic-block instruction counts from an ncu report's SASS source page.
usage: sass_blocks.py rep.ncu-rep units [top]   (units = e.g. slices, to print per-unit counts)"""
import csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2]); top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]; ie = h.index("Instructions Executed")
rows = r[2:]
tot = sum(int(x[ie]) for x in rows if x[ie].isdigit())
print(f"total {tot}  per unit {tot / units:.1f}")
blocks = []
for x in rows:
    e = int(x[ie]) if x[ie].isdigit() else 0
    if blocks and blocks[-1][1] == e:
        blocks[-1][2] += 1; blocks[-1][3].append(x[1].strip())
    else:
        blocks.append([x[0], e, 1, [x[1].strip()]])
for b in sorted(blocks, key=lambda b: -b[1] * b[2])[:top]:
    print(f"{b[0][-5:]} exec={b[1]:>11d} n={b[2]:>3d} per-unit={b[1] * b[2] / units:6.1f} | " + " | ".join(b[3][:5])[:140])
