"""Static SASS loop bodies of one kernel (backward branches), with an opcode histogram.

usage: sass_loops.py MANGLED_SUBSTRING [cubin-name-prefix | path.cubin]
Disassembles the in-tree libfvv_b200.so."""
import collections
import os
import re
import subprocess
import sys
import tempfile

name = sys.argv[1]
prefix = sys.argv[2] if len(sys.argv) > 2 else "interp_kernels"
if prefix.endswith(".cubin"):  # a cubin built by hand (e.g. nvcc -cubin -D... for a variant)
    cubp = prefix
else:
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath("paper_2112_10603_b200/libfvv_b200.so")], cwd=tmp,
                   capture_output=True)
    cubp = os.path.join(tmp, [f for f in os.listdir(tmp) if f.startswith(prefix) and f.endswith(".cubin")][0])
dis = subprocess.run(["nvdisasm", "-c", cubp], capture_output=True, text=True).stdout
i = dis.index(".text." + name)
j = dis.find("//-----", i + 10)
sec = dis[i:j].split("\n")
ins, labels = [], {}
for l in sec:
    m = re.match(r"\s*(\.L_x_\d+):", l)
    if m:
        labels[m.group(1)] = len(ins)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append(m.group(2).strip())
print(f"{len(ins)} instructions")
for k, t in enumerate(ins):
    m = re.search(r"BRA.*`\((\.L_x_\d+)\)", t)
    if m and labels.get(m.group(1), 1 << 30) <= k:
        body = ins[labels[m.group(1)]:k + 1]
        c = collections.Counter(x.split()[1] if x.startswith("@") else x.split()[0] for x in body)
        print(f"loop {labels[m.group(1)]}..{k} ({len(body)} instr):", dict(c.most_common(12)))
