"""RefineNet + ContextNet on the cfg4 rig (7 pairs x 15 views, 1080p YUV420): one
warm-up and one measured pass (for ncu launch lists: tools/launch_summary.py)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from bench import synth_rig  # noqa: E402
from paper_2112_10603_b200.refine import RefineNet  # noqa: E402
from paper_2112_10603_b200.vinet import VINet  # noqa: E402

W, H, fmt, C, nv = 1920, 1080, 1, 8, 15
cams = torch.from_numpy(synth_rig(W, H, fmt, C)).cuda()
L, R = cams[:-1].contiguous(), cams[1:].contiguous()
net = VINet(W, H, fmt, max_pairs=C - 1)
flows = net.flows(L, R)
ref = RefineNet(W, H, fmt, max_views=nv)
out = ref.views(L, R, flows, nv)
torch.cuda.synchronize()
t = time.perf_counter()
ref.views(L, R, flows, nv, out=out)
torch.cuda.synchronize()
print(f"refine {1e3 * (time.perf_counter() - t):.1f} ms (host-timed, eager)")
