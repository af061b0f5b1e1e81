"""Quick VINet timing: flows (+ synth) for a batch of 1080p pairs; conv TFLOP/s."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2112_10603_b200.vinet import VINet  # noqa: E402
from paper_2112_10603_b200.vinet_params import BLOCK_IN  # noqa: E402


def conv_flops(W, H):
    Wp, Hp = (W + 63) // 64 * 64, (H + 63) // 64 * 64
    tot = 0
    for i in range(3):
        w, h = Wp >> (2 - i), Hp >> (2 - i)
        cin = BLOCK_IN[i]
        tot += 2 * (w // 2) * (h // 2) * 128 * 9 * cin          # c0
        tot += 2 * (w // 4) * (h // 4) * 256 * 9 * 128          # c1
        tot += 6 * 2 * (w // 4) * (h // 4) * 256 * 9 * 256      # r1..r6
        tot += 2 * (w // 2) * (h // 2) * 128 * 4 * 256          # u0 (4 taps per output)
        tot += 2 * w * h * 5 * 4 * 128                          # u1
    return tot


W, H, fmt = int(sys.argv[1]) if len(sys.argv) > 1 else 1920, int(sys.argv[2]) if len(sys.argv) > 2 else 1080, 1
npairs = int(sys.argv[3]) if len(sys.argv) > 3 else 7
nviews = 15
fb = W * H * 3 // 2
net = VINet(W, H, fmt, max_pairs=npairs)
rng = np.random.default_rng(0)
L = torch.from_numpy(rng.integers(0, 256, (npairs, fb), dtype=np.uint8)).cuda()
R = torch.roll(L, 3, 1)
if len(sys.argv) > 4 and sys.argv[4] == "rig2":  # two fused rig frames only (ncu launch lists: keep the 2nd)
    cams = torch.cat([L, R[-1:]], 0).contiguous()
    for _ in range(2):
        net.rig_clusters(cams, 4, 16)
    torch.cuda.synchronize()
    sys.exit(0)
fl = net.flows(L, R)
views = net.synth(L, R, fl, nviews)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
K = 10
ev[0].record()
for _ in range(K):
    net.flows(L, R, out=fl)
ev[1].record()
for _ in range(K):
    net.synth(L, R, fl, nviews, out=views)
ev[2].record()
torch.cuda.synchronize()
tf = ev[0].elapsed_time(ev[1]) / K
ts = ev[1].elapsed_time(ev[2]) / K
fl_ = conv_flops(W, H) * npairs
print(f"{W}x{H} pairs {npairs}: flows {tf:.2f} ms ({fl_ / tf / 1e9:.0f} TFLOP/s conv-equivalent, "
      f"{fl_ / 1e12:.2f} TFLOP), synth {nviews} views {ts:.2f} ms -> "
      f"{npairs * nviews / ((tf + ts) / 1e3):.0f} views/s")

# the fused rig path (flows + synthesis with the cluster tiles in its epilogue + anchors/padding)
cams = torch.cat([L, R[-1:]], 0).contiguous()
views, cl, _ = net.rig_clusters(cams, 4, 16)
torch.cuda.synchronize()
ev[0].record()
for _ in range(K):
    net.rig_clusters(cams, 4, 16, views=views, out=cl)
ev[1].record()
torch.cuda.synchronize()
print(f"rig_clusters (8 cams, 4 stages, vps 16): {ev[0].elapsed_time(ev[1]) / K:.2f} ms")
from paper_2112_10603_b200.cluster import rig_clusters  # noqa: E402
ev[0].record()
for _ in range(K):
    net.rig(cams, 4, views=views)
    rig_clusters(views, W, H, fmt, cams.shape[0], 4, 16, out=cl)
ev[1].record()
torch.cuda.synchronize()
print(f"rig + rig_clusters, unfused: {ev[0].elapsed_time(ev[1]) / K:.2f} ms")
