"""Aggregate an ncu SASS source page by CUDA source line.

usage: stall_by_line.py REPORT KERNEL_SUBSTR MANGLED_NAME [top]
The line table comes from nvdisasm -g on the in-tree libfvv_b200.so (must be
the binary that was profiled)."""
import collections
import csv
import re
import subprocess
import sys
import tempfile
import os

rep, ksub, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
secs, cur, hdr = [], None, None
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = [x[1], [], None]
        secs.append(cur)
        continue
    if x and x[0] == "Address":
        cur[2] = x
        continue
    if cur and len(x) > 5:
        cur[1].append(x)
body, hdr = [(b, h) for n, b, h in secs if ksub in n][0]
col = {k: hdr.index(k) for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)", "stall_long_sb",
                                 "stall_short_sb", "stall_wait", "stall_math", "stall_not_selected")}
base = int(body[0][0], 16)

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath("paper_2112_10603_b200/libfvv_b200.so")], cwd=tmp,
               capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("interp_kernels") and f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
i = dis.index(".text." + mangled + ":")
j = dis.find("\t.section", i + 10)
dis = dis[i:j if j > 0 else len(dis)]
line_of = {}
cur_line = None
for l in dis.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if "//##" in l and m:
        cur_line = os.path.basename(m.group(1)).split(".")[0][:6] + ":" + m.group(2)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur_line is not None:
        line_of[int(m.group(1), 16)] = cur_line
agg = collections.defaultdict(lambda: collections.Counter())
for x in body:
    off = int(x[0], 16) - base
    ln = line_of.get(off, "?")
    for k, i in col.items():
        try:
            agg[ln][k] += float(x[i] or 0)
        except ValueError:
            pass
tot = {k: sum(a[k] for a in agg.values()) or 1 for k in col}
print("         line   inst%  samples%  long_sb%  short_sb%  wait%")
for ln, a in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    print(f"{ln:>13} {a['Instructions Executed'] / tot['Instructions Executed'] * 100:6.1f} "
          f"{a['Warp Stall Sampling (All Samples)'] / tot['Warp Stall Sampling (All Samples)'] * 100:8.1f} "
          f"{a['stall_long_sb'] / tot['stall_long_sb'] * 100:8.1f} {a['stall_short_sb'] / tot['stall_short_sb'] * 100:8.1f}"
          f" {a['stall_wait'] / tot['stall_wait'] * 100:6.1f}")
