"""Aggregate an ncu source page by kernel phase: every source line of
small_tree.cu is assigned to the last '// ---------------- (x)' phase marker
above it (other files count as 'helpers').

  python profiles/ncu_phases.py report.ncu-rep [path/to/small_tree.cu]
"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_2001_07104_b200/csrc/small_tree.cu"
marks = []
for i, line in enumerate(open(src), 1):
    m = re.search(r"// -{4,} \((\w)\) (.*)", line)
    if m:
        marks.append((i, f"({m.group(1)}) {m.group(2)[:40]}"))
    elif "// ---- " in line:
        marks.append((i, line.strip()[8:48]))


def phase(ln):
    name = "prologue"
    for i, nm in marks:
        if i <= ln:
            name = nm
    return name


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0])
cur, hdr = None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))
    key = phase(ln) if cur == "small_tree.cu" else "helpers (" + str(cur) + ")"
    agg[key][0] += float(d.get("Instructions Executed", "0") or 0)
    agg[key][1] += float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total inst {ti:.3e}  stall samples {ts:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:50s} inst {100 * v[0] / ti:5.1f}%  samples {100 * v[1] / ts:5.1f}%")
