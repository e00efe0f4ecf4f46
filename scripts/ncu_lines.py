"""Per-CUDA-source-line instruction and stall attribution from an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []; fname = None; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or not r[0].isdigit(): continue
    try:
        st = float(r[4]); ex = float(r[7])
    except ValueError:
        continue
    res.append((ex, st, fname, int(r[0]), r[1][:90]))
tex = sum(x[0] for x in res); tst = sum(x[1] for x in res)
for ex, st, f, ln, src in sorted(res, key=lambda x: -x[0])[:topn]:
    print(f"{100*ex/tex:5.1f}% instr {100*st/tst:5.1f}% stall  {f}:{ln:4d}  {src}")
