"""Top source lines of one kernel in an ncu report by warp-stall samples
(--import-source on).  usage: ncu_stall_lines.py report [launch_index] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, fname, cur, tot = {}, None, None, 0
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:70])
        continue
    if r[2].startswith("0x") and cur:
        try:
            s = int(r[4])
        except ValueError:
            continue
        agg[cur] = agg.get(cur, 0) + s
        tot += s
print(f"stall samples: {tot}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100.0 * v / max(1, tot):5.1f}%  {k[0]}:{k[1]}  {k[2]}")
