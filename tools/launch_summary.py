"""Summarise an ncu launch list (CSV of gpu__time_duration / smsp__inst_executed /
dram__bytes_read / dram__bytes_write per launch) into a markdown table and the
per-pair traffic table bench.py reads (profiles/traffic.json).

usage: launch_summary.py LAUNCHES_CSV TAG CONFIG [--traffic profiles/traffic.json] [--md OUT.md]
"""
import argparse
import collections
import csv
import json
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("tag")
ap.add_argument("config")
ap.add_argument("--traffic")
ap.add_argument("--md")
a = ap.parse_args()

rows = [r for r in csv.reader(open(a.csv)) if len(r) > 12 and r[0].isdigit()]
launch = collections.defaultdict(dict)
for r in rows:
    lid, name, grid, metric, val = int(r[0]), r[4], r[8], r[12], r[14]
    launch[lid]["name"] = name
    launch[lid]["grid"] = tuple(int(v) for v in re.findall(r"\d+", grid))
    launch[lid][metric] = float(val.replace(",", ""))


def short(name):
    n = re.sub(r"^void ", "", name)
    return re.sub(r"\(.*$", "", n)


def kclass(name):
    s = short(name)
    m = re.match(r"fvv::k_sad\w*<(\d)", s)
    if m:
        return f"k_sad<{m.group(1)}>"
    m = re.match(r"fvv::(k_warpq|k_flow)<(\d)", s)
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    m = re.match(r"fvv::(k_pyramid|k_mask_cols|k_scan_carry|k_blend|k_rig_clusters|k_sd)(?:2)?\b", s)
    return m.group(1) if m else None


def pairs(name, grid):
    s = short(name)
    if any(k in s for k in ("k_sad", "k_flow", "k_warpq", "k_pyramid")):
        return grid[2] // 2
    if "k_scan_carry" in s:
        return grid[1]
    if any(k in s for k in ("k_mask_cols", "k_blend", "k_sd")):
        return grid[2]
    return 0


agg = collections.defaultdict(lambda: collections.Counter())
tot_t = 0.0
for l in launch.values():
    if "gpu__time_duration.sum" not in l:
        continue
    key = short(l["name"])
    c = agg[key]
    c["n"] += 1
    c["t"] += l["gpu__time_duration.sum"]
    c["inst"] += l.get("smsp__inst_executed.sum", 0)
    c["dram"] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    c["pairs"] += pairs(l["name"], l["grid"])
    c["cls"] = 0
    tot_t += l["gpu__time_duration.sum"]
names = {short(l["name"]): l["name"] for l in launch.values()}
lines = [f"| kernel | launches | interp pairs | time share | warp-instr per pair (M) | DRAM read+write per pair (MB) |",
         "|---|---|---|---|---|---|"]
traffic = {}
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
    p = c["pairs"]
    ipp = f"{c['inst'] / p / 1e6:.2f}" if p else "-"
    dpp = f"{c['dram'] / p / 1e6:.1f}" if p else "-"
    lines.append(f"| {key} | {c['n']} | {p or '-'} | {c['t'] / tot_t:.3f} | {ipp} | {dpp} |")
    cls = kclass(names[key])
    if cls and p:
        t = traffic.setdefault(cls, {"warp_inst_per_pair": 0.0, "dram_bytes_per_pair": 0.0, "source": []})
        t["warp_inst_per_pair"] += c["inst"] / p
        t["dram_bytes_per_pair"] += c["dram"] / p
        t["source"].append(key)
for t in traffic.values():
    t["source"] = f"ncu launch list {a.tag} (" + " + ".join(t["source"]) + ")"
md = "\n".join(lines)
print(md)
if a.md:
    with open(a.md, "w") as f:
        f.write(f"# {a.tag} -- ncu launch list, {a.config}\n\n"
                "`ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,"
                "dram__bytes_write.sum --clock-control none` over `bench.py --steps 2 --warmup 1` -- cold "
                "cache, serialised: compare shares, not absolute times.\n\n" + md + "\n")
if a.traffic:
    try:
        allt = json.load(open(a.traffic))
    except OSError:
        allt = {}
    allt[a.config] = traffic
    json.dump(allt, open(a.traffic, "w"), indent=1)
