"""Per-source-line dynamic SASS mix of one kernel in an ncu report
(--import-source on): instructions per output point and top opcodes.
usage: sass_lines.py report.ncu-rep points [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, npts = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30


def page(src):
    return list(csv.reader(io.StringIO(subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", src],
        capture_output=True, text=True).stdout)))


addr2line, fname, line = {}, None, None
for r in page("cuda,sass"):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        line = (fname, int(r[0]), r[1].strip()[:60])
    if len(r) > 2 and r[2].startswith("0x"):
        addr2line[r[2]] = line
rows = page("sass")
hdr = rows[1]
npw = npts / 32
ops, byline = collections.Counter(), collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    n = int(d["Instructions Executed"].replace(",", "") or 0)
    src = d["Source"].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
    ops[op] += n
    byline[addr2line.get(d["Address"])][op] += n
print(f"warp instructions per 32 points: {sum(ops.values()) / npw:.1f}")
print(" ".join(f"{o}:{c / npw:.1f}" for o, c in ops.most_common(24)))
for ln, c in sorted(byline.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    t = ", ".join(f"{o}:{v / npw:.1f}" for o, v in c.most_common(4))
    print(f"{sum(c.values()) / npw:6.2f} {ln[0]}:{ln[1]} {ln[2]:60s} | {t}")
