"""Digest of an ncu --set full report for profiles/: headline metrics, DRAM bytes, fp64 pipe
instructions, stall mix and the hottest source lines.

  python profiles/ncu_digest.py gpurun_out/<rep>.ncu-rep [top_lines]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def page(name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


det = page("details")
hdr = det[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Registers Per Thread", "Theoretical Active Warps per SM",
        "Achieved Active Warps Per SM", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Branch Efficiency", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]
for row in det[1:]:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:36s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = page("raw")
h, units, vals = raw[0], raw[1], raw[2]
d = dict(zip(h, vals))
u = dict(zip(h, units))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__inst_executed.sum",
          "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed_pipe_fp64.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
          "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]:
    if k in d:
        print(f"{k:60s} {d[k]:>18s} {u.get(k, '')}")
st = {k: num(k) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(v for v in st.values() if v) or 1
print("stall samples (top):")
for k, v in sorted(st.items(), key=lambda kv: -(kv[1] or 0))[:8]:
    if v:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f} %")
src = page("source", ("--print-source=cuda,sass",))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
cur = None
shdr = None
for r in src:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        shdr = r
        continue
    if shdr is None:
        continue
    dd = dict(zip(shdr, r))
    try:
        line = int(r[0])
        agg[(cur, line)][0] += float(dd.get("Instructions Executed", "0") or 0)
        agg[(cur, line)][1] += float(dd.get("Warp Stall Sampling (All Samples)", "0") or 0)
        agg[(cur, line)][2] = r[1][:90]
    except ValueError:
        pass
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print("hottest source lines (share of instructions / stall samples):")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {k[0][:14]:14s}:{k[1]:5d}  inst {100 * v[0] / ti:5.1f} %  stall {100 * v[1] / ts:5.1f} %  {v[2]}")
