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
