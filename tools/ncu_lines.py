"""Aggregate ncu warp-stall samples per CUDA source line.

    python tools/ncu_lines.py report.ncu-rep [kernel-substring] [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
col = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"  # or "Instructions Executed"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
src_text = {}
fn = path = None
cur = None
si = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        fn = row[1]
        continue
    if row[0] == "Line No":
        si = row.index(col)
        continue
    if kern and (fn is None or kern not in fn):
        continue
    if row[0]:  # a source line
        cur = (path, int(row[0]))
        src_text[cur] = row[1].strip()
    if si is not None and len(row) > si and row[si] not in ("", None):
        try:
            agg[cur] += float(row[si])
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print(f"total samples {tot:.0f}")
for (k, v) in agg.most_common(top):
    print(f"{v:7.0f} {100 * v / tot:5.1f}%  {k[0]}:{k[1]}  {src_text.get(k, '')[:90]}")
