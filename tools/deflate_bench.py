"""Device DEFLATE on the cfg4 encoder's token streams (696 planes, ~83 MB):
per-call time with CUDA events; run under ncu for the per-kernel split."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import synth_rig  # noqa: E402
from paper_2112_10603_b200.cluster import build_layouts, rig_clusters  # noqa: E402
from paper_2112_10603_b200.deflate import deflate_streams  # noqa: E402
from paper_2112_10603_b200.encoder import RigEncoder  # noqa: E402
from paper_2112_10603_b200.interp import Interpolator  # noqa: E402
from paper_2112_10603_b200.viewmodel import ViewIndexModel  # noqa: E402

W, H, C, S, vps = 1920, 1080, 8, 4, 16
eng = Interpolator(W, H, 1, max_pairs=56)
cams = torch.from_numpy(synth_rig(W, H, 1, C, seed=42)).cuda()
views = eng.rig(cams, S)
buf = rig_clusters(views, W, H, 1, C, S, vps)[0].clone()
enc = RigEncoder(build_layouts(ViewIndexModel(C, S), vps), W, H, 1, quality=75, gop=30, threads=16)
enc.encode(buf)
offs = enc.tok_off[:enc.nblocks + 1].cpu().numpy()
jobs = enc._last_jobs.cpu().numpy().view(np.int64).reshape(-1, 8)
plane_offs = [0]
for j in enc._last_jobs.cpu().numpy().view(np.uint8).reshape(-1, 64):
    b0 = int(j[24:32].view(np.int64)[0])
    nbx, nby = int(j[44:48].view(np.int32)[0]), int(j[48:52].view(np.int32)[0])
    plane_offs.append(int(offs[b0 + nbx * nby]) * 3)
tok = enc.tokens[:plane_offs[-1]]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for _ in range(2):
    deflate_streams(tok, plane_offs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    out, oo = deflate_streams(tok, plane_offs)
e1.record()
torch.cuda.synchronize()
print(f"device deflate: {len(plane_offs) - 1} streams, {plane_offs[-1] / 1e6:.1f} MB -> "
      f"{int(oo[-1]) / 1e6:.1f} MB in {e0.elapsed_time(e1) / reps:.2f} ms per call")
if len(sys.argv) > 2:  # dump the largest and a median plane stream for the host model
    sizes = np.diff(plane_offs)
    order = np.argsort(sizes)
    host = tok.cpu().numpy()
    for tag, i in (("largest", int(order[-1])), ("median", int(order[len(order) // 2]))):
        host[plane_offs[i]:plane_offs[i + 1]].tofile(f"{sys.argv[2]}/tok_{tag}.bin")
