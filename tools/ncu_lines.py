"""Per-source-line attribution of an ncu capture (stall samples, warp
instructions) by joining the SASS page with nvdisasm line info:
    python tools/ncu_lines.py <rep.ncu-rep> <obj.o> <mangled kernel name> [topN] [outer|inner|full]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
mode = sys.argv[5] if len(sys.argv) > 5 else "outer"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
addr2line, cur, on, cur_pending = {}, None, False, True
for ln in dis.splitlines():
    if ln.startswith(".text."):
        on = ln.strip().rstrip(":") == ".text." + fn
        continue
    if not on:
        continue
    if "//## File" in ln:
        locs = re.findall(r'"([^"]+)", line (\d+)', ln)
        if cur_pending:
            cur = " < ".join(f"{os.path.basename(f)}:{l}" for f, l in locs)
            cur_pending = False
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        addr2line[int(m.group(1), 16)] = cur
        cur_pending = True
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
st, ins, exc = collections.Counter(), collections.Counter(), collections.Counter()
base = None
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else int(r[ix["Address"]])
    base = a if base is None else base
    line = addr2line.get(a - base, "?")
    if mode == "outer":
        line = line.split(" < ")[-1]
    elif mode == "inner":
        line = line.split(" < ")[0]
    st[line] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ins[line] += float(r[ix["Instructions Executed"]] or 0)
    try:
        exc[line] += float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    except (KeyError, ValueError):
        pass
ts, ti, te = sum(st.values()), sum(ins.values()), max(sum(exc.values()), 1)
print(f"{'line':40s} {'stall%':>7s} {'inst%':>7s} {'smem-excess%':>12s}")
for line, s in st.most_common(top):
    print(f"{line:40s} {s / ts * 100:7.2f} {ins[line] / ti * 100:7.2f} {exc[line] / te * 100:12.2f}")
