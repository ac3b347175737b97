"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

  python profiles/launch_share.py gpurun_out/<tag>_launches.csv [skip_first_n]

ncu times are cold-cache and serialised: compare the SHARES with bench.py's
kernels_ms_per_step, not the absolute numbers."""
import collections
import csv
import re
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr = rows[0]
recs = [dict(zip(hdr, r)) for r in rows[1:]]
recs = [r for r in recs if r["Metric Name"] == "gpu__time_duration.sum"][skip:]
agg = collections.defaultdict(lambda: [0.0, 0])
for r in recs:
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("rf::<unnamed>::", "")
    agg[name][0] += float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
    agg[name][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"# {len(recs)} launches, {tot / 1e3:.3f} ms total device time (ncu, serialised)")
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k[:60]:60s} {v[1]:8d} {v[0]:12.1f} {100 * v[0] / tot:6.2f}%")
