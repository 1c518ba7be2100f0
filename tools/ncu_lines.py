"""Per-source-line instruction and stall attribution from an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, lines, fname = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr[2:], r[2:]))
        def num(k):
            v = (d.get(k) or "0").replace(",", "")
            return int(v) if v.isdigit() else 0
        lines.append((num("Instructions Executed"), num("Warp Stall Sampling (All Samples)"), fname,
                      r[0], r[1]))
tot = sum(l[0] for l in lines) or 1
tst = sum(l[1] for l in lines) or 1
print(f"warp instructions {tot}, stall samples {tst}")
for ie, st, f, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{100*ie/tot:5.1f}% i {100*st/tst:5.1f}% s {f}:{ln}: {src.strip()[:88]}")
