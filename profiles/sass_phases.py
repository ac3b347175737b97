"""Per-phase instruction and stall split of the small-tree kernel from an ncu capture.

  python profiles/sass_phases.py <report.ncu-rep> [kernel-variant-substring]

Maps every SASS instruction to a phase of small_tree.cu through its kernel-body source line
(nvdisasm -gi: the line an inlined helper was inlined at), the phases being delimited by the
PT_MARK(i) markers of the source (the same phases as the RF_PHASE_TIMING build), then sums
ncu's per-instruction "Instructions Executed" and warp-stall samples per phase.  Unlike the
phase-timing build (warp cycles, latency included) this gives the issued-instruction share.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "..", "paper_2001_07104_b200", "csrc", "small_tree.cu")
OBJ = os.path.join(HERE, "..", "build", "small_tree.o")
NAMES = {0: "tree setup (bootstrap, root, in-bag lists)", 1: "(a) node prefixes", 2: "(a) feature draws",
         3: "(a) ExtraTrees thresholds", 4: "(b) search pass 1 + scan", 5: "(b) search pass 2 + node bests",
         6: "(c) decide", 7: "(d) mark", 8: "(e) children / emission", 9: "(f) test-row routing",
         10: "(g) partition list 0", 11: "(g) partition lists 1..p-1", 12: "level advance", 13: "tree end",
         14: "CTA prologue", 15: "epilogue"}


def phase_of_line():
    marks = []
    for no, line in enumerate(open(SRC), 1):
        m = re.search(r"PT_MARK\((\d+)\);", line)
        if m and "define" not in line:
            marks.append((no, int(m.group(1))))
    marks.sort()

    def f(line):
        for no, ph in marks:
            if line <= no:
                return ph
        return 15
    return f, marks[0][0] - 120  # kernel body starts ~ before the first mark


def sass_lines(variant):
    import tempfile
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", OBJ], cwd=tmp, check=True, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    addr_line = {}
    cur_fun = None
    line = inl = None
    for ln in out.splitlines():
        m = re.match(r"^(_Z\S+):$", ln)
        if m:
            cur_fun = m.group(1)
            continue
        m = re.search(r'//## File ".*small_tree\.cu", line (\d+)(?: inlined at ".*?", line (\d+))?', ln)
        if m:
            line = int(m.group(1))
            inl = int(m.group(2)) if m.group(2) else None
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fun and variant in cur_fun and line is not None:
            addr_line[int(m.group(1), 16)] = (line, inl)
    return addr_line


def main():
    rep = sys.argv[1]
    variant = sys.argv[2] if len(sys.argv) > 2 else "small_tree_kernelILb0ELi1ELb0ELb0E"
    ph, body0 = phase_of_line()
    amap = sass_lines(variant)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = None
    base = None  # the report's addresses are absolute: offsets from the function's first instruction
    inst = collections.Counter()
    stall = collections.Counter()
    for r in rows:
        if r and r[0] in ("Address", "# Address"):
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            a = int(d.get("Address", d.get("# Address", "")), 16)
        except ValueError:
            continue
        if base is None:
            base = a
        li = amap.get(a - base)
        if li is None:
            continue
        line, inl = li
        body = line if (line >= body0 or inl is None) else inl
        p = ph(body) if body >= body0 else 15
        inst[p] += float(d.get("Instructions Executed", 0) or 0)
        stall[p] += float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
    ti, ts = sum(inst.values()), sum(stall.values())
    print(f"total {ti:.4e} warp instructions, {ts:.4e} stall samples")
    for p in sorted(inst, key=lambda k: -inst[k]):
        print(f"  {NAMES.get(p, p):44s} inst {100 * inst[p] / ti:5.1f} %   stall {100 * stall[p] / max(ts, 1):5.1f} %")


if __name__ == "__main__":
    main()
