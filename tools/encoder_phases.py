"""Wall-time split of RigEncoder.encode on the cfg4 rig frame (P tick)."""
import cProfile
import pstats
import sys
import time

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
for seed in (42, 4242, 7):
    cams = torch.from_numpy(synth_rig(W, H, 1, C, seed=seed)).cuda()
    bufs.append(rig_clusters(eng.rig(cams, S), W, H, 1, C, S, vps)[0].clone())
enc = RigEncoder(build_layouts(ViewIndexModel(C, S), vps), W, H, 1, quality=75, gop=30, threads=16)
enc.encode(bufs[0])
enc.encode(bufs[1])
torch.cuda.synchronize()
t = time.perf_counter()
enc.encode(bufs[2])
print(f"encode wall {1e3 * (time.perf_counter() - t):.1f} ms")
pr = cProfile.Profile()
pr.enable()
enc.encode(bufs[1])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
