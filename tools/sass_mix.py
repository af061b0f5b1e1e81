"""Summarise an ncu report: per kernel metrics + executed-instruction mix (SASS)."""
import csv
import collections
import subprocess
import sys

rep = sys.argv[1]
mets = ("gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,"
        "sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,"
        "smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,"
        "dram__bytes_read.sum,dram__bytes_write.sum")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", mets],
                     capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
for row in r[2:]:
    print(row[4][:60])
    print("   ", ", ".join(f"{h[i].split('.')[0].replace('__', ':')}={row[i]}" for i in range(11, len(h))))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
secs, cur, hdr = [], None, None
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = [x[1], []]
        secs.append(cur)
        continue
    if x and x[0] == "Address":
        hdr = x
        continue
    if cur and len(x) > 5:
        cur[1].append(x)
ie = hdr.index("Instructions Executed")
seen = set()
for name, body in secs:
    if name in seen:
        continue
    seen.add(name)
    tot = sum(int(x[ie]) for x in body)
    ops = collections.Counter()
    for x in body:
        t = x[1].strip().split()
        ops[t[1] if t[0].startswith("@") else t[0]] += int(x[ie])
    print(name[:70], tot)
    print("   ", ", ".join(f"{o} {c / tot * 100:.1f}%" for o, c in ops.most_common(16)))
