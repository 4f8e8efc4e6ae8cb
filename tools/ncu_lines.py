"""Per-source-line summary of an ncu report (--print-source cuda,sass):
python tools/ncu_lines.py report.ncu-rep [top]  -> samples, instructions,
avg threads per executed instruction, per CUDA line, sorted by samples."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for rec in csv.reader(io.StringIO(txt)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("Function Name",):
        continue
    if rec[2] != "-":  # sass rows carry an address; line rows have "-"
        continue
    d = dict(zip(hdr[2:], rec[2:]))
    try:
        samp = int(d["Warp Stall Sampling (All Samples)"])
        inst = int(d["Instructions Executed"])
        thr = int(d["Thread Instructions Executed"])
    except (KeyError, ValueError):
        continue
    rows.append((samp, inst, thr, fname, rec[0], rec[1].strip()[:90]))
ts = sum(r[0] for r in rows) or 1
ti = sum(r[1] for r in rows) or 1
print(f"total samples {ts} instructions {ti}")
for s, i, t, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{f[:12]:12s} {ln:>4s} {100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst {t/max(i,1):5.1f} thr  {src}")
