"""Phase timing of encoder.RigEncoder on the cfg4 rig frame (device transform, token D2H, host DEFLATE)."""
import sys
import time
import zlib

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import synth_rig  # noqa: E402
from paper_2112_10603_b200.cluster import build_layouts, rig_clusters  # noqa: E402
from paper_2112_10603_b200.encoder import RigEncoder  # noqa: E402
from paper_2112_10603_b200.interp import Interpolator  # noqa: E402
from paper_2112_10603_b200.viewmodel import ViewIndexModel  # noqa: E402

W, H, C, S, vps = 1920, 1080, 8, 4, 16
eng = Interpolator(W, H, 1, max_pairs=56)
bufs = []
for seed in (42, 4242):
    cams = torch.from_numpy(synth_rig(W, H, 1, C, seed=seed)).cuda()
    views = eng.rig(cams, S)
    bufs.append(rig_clusters(views, W, H, 1, C, S, vps)[0].clone())
torch.cuda.synchronize()
enc = RigEncoder(build_layouts(ViewIndexModel(C, S), vps), W, H, 1, quality=75, gop=30, threads=16)
enc.encode(bufs[0])
t = time.perf_counter()
recs = enc.encode(bufs[1])
print(f"encode (P) wall {1e3 * (time.perf_counter() - t):.1f} ms, out {sum(len(r) for c in recs for r in c) / 1e6:.1f} MB")
# token bytes and single-thread deflate cost of the largest plane
offs = enc.tok_off[:enc.nblocks + 1].cpu().numpy()
tok = enc.tokens[:int(offs[-1]) * 3].cpu().numpy().tobytes()
print(f"tokens {len(tok) / 1e6:.1f} MB over {enc.nblocks} blocks")
t = time.perf_counter()
z = zlib.compress(tok, 6)
dt = time.perf_counter() - t
print(f"zlib level 6 single thread on all tokens: {1e3 * dt:.0f} ms ({len(tok) / dt / 1e6:.0f} MB/s) -> {len(z) / 1e6:.1f} MB")
import os
print("cpus", os.cpu_count())
# per-plane DEFLATE cost: the longest single stream bounds any host schedule
sizes, times = [], []
for m in range(enc.nblocks and len(enc._last_jobs) // 64 or 0):
    pass
import heapq
meta_b = []
jobs = enc._last_jobs.cpu().numpy().view(np.dtype([("src", "<u8"), ("prev", "<u8"), ("recon", "<u8"), ("block0", "<i8"), ("pitch", "<i4"), ("w", "<i4"), ("h", "<i4"), ("nbx", "<i4"), ("nby", "<i4"), ("is_p", "<i4"), ("step", "<i4"), ("pad", "<i4")]))
for j in jobs:
    b0, nb = int(j["block0"]), int(j["nbx"]) * int(j["nby"])
    seg = tok[offs[b0] * 3:offs[b0 + nb] * 3]
    t = time.perf_counter()
    zlib.compress(seg, 6)
    times.append(time.perf_counter() - t)
    sizes.append(len(seg))
times = np.array(times)
print(f"planes {len(times)}: total {1e3 * times.sum():.0f} ms single-thread, largest {1e3 * times.max():.1f} ms "
      f"({max(sizes) / 1e6:.2f} MB), median {1e3 * np.median(times):.2f} ms")
for nt in (8, 16, 32, os.cpu_count()):
    heap = [0.0] * nt
    for t in sorted(times, reverse=True):
        heapq.heapreplace(heap, heap[0] + t)
    print(f"  LPT makespan with {nt} threads: {1e3 * max(heap):.0f} ms")
# device DEFLATE of the same plane streams: time and identity
from paper_2112_10603_b200.deflate import deflate_streams  # noqa: E402
tokdev = enc.tokens[:int(offs[-1]) * 3]
plane_offs = [0]
for j in jobs:
    b0, nb = int(j["block0"]), int(j["nbx"]) * int(j["nby"])
    plane_offs.append(int(offs[b0 + nb]) * 3)
for _ in range(2):
    out, oo = deflate_streams(tokdev, plane_offs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    out, oo = deflate_streams(tokdev, plane_offs)
e1.record()
torch.cuda.synchronize()
print(f"device deflate of {len(plane_offs) - 1} plane streams ({len(tok) / 1e6:.1f} MB): {e0.elapsed_time(e1) / 5:.2f} ms")
oo = oo.cpu().numpy()
raw = out[:int(oo[-1])].cpu().numpy().tobytes()
mism = sum(raw[oo[i]:oo[i + 1]] != zlib.compress(tok[plane_offs[i]:plane_offs[i + 1]], 6)[2:-4] for i in range(len(plane_offs) - 1))
print(f"device deflate vs zlib: {mism} of {len(plane_offs) - 1} streams differ")
