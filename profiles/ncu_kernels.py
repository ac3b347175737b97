"""One line per captured kernel of an ncu report (--set full): duration, DRAM bytes and
throughput, occupancy, IPC and the top stall reasons.

  python profiles/ncu_kernels.py report.ncu-rep
"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}
for row in rows[2:]:
    d = dict(zip(h, row))
    u = dict(zip(h, units))

    def val(k):
        v = float(d[k].replace(",", ""))
        return v * scale.get(u[k], 1)

    ms = val("gpu__time_duration.sum")
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and v.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
    name = d["Kernel Name"].split("(")[0].replace("rf::<unnamed>::", "")
    print(f"{name}: {ms:.3f} ms, DRAM read {rd / 1e9:.3f} GB + write {wr / 1e9:.3f} GB = "
          f"{(rd + wr) / (ms * 1e-3) / 1e9:.0f} GB/s, warps active "
          f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.0f} %, regs "
          f"{d['launch__registers_per_thread']}, IPC {float(d['sm__inst_executed.avg.per_cycle_active']):.2f}; "
          f"stalls: {top}")
