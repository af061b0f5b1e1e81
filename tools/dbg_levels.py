"""Debug helper: per-level flow / match-error comparison against a golden file."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
from conftest import load_golden
from paper_2112_10603_b200.interp import Interpolator

name = sys.argv[1] if len(sys.argv) > 1 else "scene_gray8_64x48"
g = load_golden(name)
w, h, fmt = int(g["w"]), int(g["h"]), int(g["fmt"])
eng = Interpolator(w, h, fmt, None, max_pairs=1)
out = eng.pairs(torch.from_numpy(g["left"][None]).cuda(), torch.from_numpy(g["right"][None]).cuda())
torch.cuda.synchronize()
print(name, "out bytes differ:", int(np.count_nonzero(out.cpu().numpy()[0] != g["out"])))
for s in range(3):
    if f"lv{s}_flow_lr" not in g:
        continue
    flr, frl, elr, erl = eng.level_diagnostics(0, s)
    for k, v in (("flow_lr", flr), ("flow_rl", frl), ("err_lr", elr), ("err_rl", erl)):
        ref = g[f"lv{s}_{k}"]
        got = v.cpu().numpy()
        bad = np.argwhere(got != ref)
        print(f"  level {s} {k}: {len(bad)} mismatches", bad[:3].tolist(),
              [got[tuple(b)] for b in bad[:3]], [ref[tuple(b)] for b in bad[:3]])
