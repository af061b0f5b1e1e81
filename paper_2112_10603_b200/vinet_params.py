"""VINet architecture constants and its seeded parameter set (no compute here).

VINet ("View Interpolation Network", layer table
PAPER.md:320-337): three VIBlocks estimate the mid-view flows and the fusion
mask coarse to fine, RIFE-style (the paper cites RIFE).  The reference
package ships no CNN, so this module pins the architecture the
north star names and a deterministic random initialisation; the fp32 torch
oracle (oracle/vinet_ref.py) and the B200 engine (vinet.py) both read the
same tensors from here.

VIBlock_i (i = 0, 1, 2) works at r_i = 2^i / 4 of the input resolution:
  c0  Conv2d 3x3 s2  cin -> 128, ReLU            (r_i / 2)
  c1  Conv2d 3x3 s2  128 -> 256, ReLU            (r_i / 4)
  r1..r6  Conv2d 3x3 s1  256 -> 256, ReLU        (r_i / 4)
  u0  ConvTranspose2d 4x4 s2 p1  256 -> 128, ReLU (r_i / 2)
  u1  ConvTranspose2d 4x4 s2 p1  128 -> 5         (r_i): residual of
      (F_m->l.x, F_m->l.y, F_m->r.x, F_m->r.y, mask logit), flows in pixels of r_i.
Inputs: block 0 = (I_l, I_r) at r_0 (6 ch); blocks 1, 2 = (I_l, I_r,
warp(I_l, F_l), warp(I_r, F_r), F_l, F_r, M) at r_i (17 ch), with F, M the
previous estimate upsampled 2x (flows times 2).  Images are 3 channels in
[0, 1]: RGB, or (Y, U, V) with chroma repeated 2x2, or (Y, 0.5, 0.5).
"""
from __future__ import annotations

BLOCK_IN = (6, 17, 17)
LAYERS = (  # name, kind, cin, cout
    ("c0", "conv_s2", None, 128),
    ("c1", "conv_s2", 128, 256),
    ("r1", "conv", 256, 256), ("r2", "conv", 256, 256), ("r3", "conv", 256, 256),
    ("r4", "conv", 256, 256), ("r5", "conv", 256, 256), ("r6", "conv", 256, 256),
    ("u0", "convT", 256, 128),
    ("u1", "convT", 128, 5),
)
HEAD_SCALE = 0.1  # the head starts small so a random network predicts flows of a few pixels


def layer_cin(block: int, k: int) -> int:
    cin = LAYERS[k][2]
    return BLOCK_IN[block] if cin is None else cin


def make_params(seed: int = 0):
    """Deterministic He-normal weights (head scaled by HEAD_SCALE), small biases.

    Returns [block][layer] = (weight, bias) as fp32 CPU tensors in torch's own
    layouts: Conv2d [cout][cin][3][3], ConvTranspose2d [cin][cout][4][4].
    """
    import torch
    g = torch.Generator().manual_seed(int(seed))
    blocks = []
    for i in range(3):
        layers = []
        for k, (name, kind, _, cout) in enumerate(LAYERS):
            cin = layer_cin(i, k)
            if kind == "convT":
                fan_in = cin * 4  # each output pixel sees 2x2 taps of cin channels
                w = torch.randn((cin, cout, 4, 4), generator=g) * (2.0 / fan_in) ** 0.5
            else:
                fan_in = cin * 9
                w = torch.randn((cout, cin, 3, 3), generator=g) * (2.0 / fan_in) ** 0.5
            if name == "u1":
                w = w * HEAD_SCALE
            b = torch.randn((cout,), generator=g) * 0.01
            layers.append((w.float(), b.float()))
        blocks.append(layers)
    return blocks


# ---------------------------------------------------------------------------
# RefineNet + ContextNet ("Refinement Network", layer table
# PAPER.md:340-365; context-aware residual U-Net after Niklaus & Liu 2018, as
# in RIFE which the paper follows).  ContextNet runs on each source image;
# after each of its 4 levels the features are backward-warped to the view
# with the level's flow (2x2 mean of the finer flow, times 0.5).  The U-Net
# input is (I_l, I_r, warp(I_l), warp(I_r), w_t, F_l,t, F_r,t) = 17 channels;
# down_k concatenates the warped context features of level k-1, the decoder
# concatenates the encoder skips; the head is conv 16 -> 3 + sigmoid and the
# view is clip(merged + 2 sigmoid - 1, 0, 1).
# ---------------------------------------------------------------------------
CONTEXT_LAYERS = (  # name, stride, cin, cout
    ("x0", 2, 3, 16), ("x1", 1, 16, 16),
    ("x2", 2, 16, 32), ("x3", 1, 32, 32),
    ("x4", 2, 32, 64), ("x5", 1, 64, 64),
    ("x6", 2, 64, 128), ("x7", 1, 128, 128),
)
CONTEXT_CH = (16, 32, 64, 128)      # warped context features per level (1/2 .. 1/16)
REFINE_IN = 17
REFINE_LAYERS = (  # name, kind, cin, cout
    ("d0a", "conv_s2", REFINE_IN, 32), ("d0b", "conv", 32, 32),
    ("d1a", "conv_s2", 32 + 2 * 16, 64), ("d1b", "conv", 64, 64),
    ("d2a", "conv_s2", 64 + 2 * 32, 128), ("d2b", "conv", 128, 128),
    ("d3a", "conv_s2", 128 + 2 * 64, 256), ("d3b", "conv", 256, 256),
    ("u0", "convT", 256 + 2 * 128, 128),
    ("u1", "convT", 128 + 128, 64),
    ("u2", "convT", 64 + 64, 32),
    ("u3", "convT", 32 + 32, 16),
    ("out", "conv", 16, 3),
)
REFINE_HEAD_SCALE = 0.1  # the residual starts small (sigmoid ~ 0.5), like the flow head


def make_refine_params(seed: int = 1):
    """Deterministic He-normal weights of ContextNet and the U-Net.

    Returns {"context": [(w, b)] * 8, "unet": [(w, b)] * 13} (fp32 CPU tensors,
    torch layouts as make_params)."""
    import torch
    g = torch.Generator().manual_seed(int(seed))

    def conv(cin, cout, scale=1.0):
        w = torch.randn((cout, cin, 3, 3), generator=g) * (2.0 / (cin * 9)) ** 0.5 * scale
        return w.float(), (torch.randn((cout,), generator=g) * 0.01).float()

    def convT(cin, cout):
        w = torch.randn((cin, cout, 4, 4), generator=g) * (2.0 / (cin * 4)) ** 0.5
        return w.float(), (torch.randn((cout,), generator=g) * 0.01).float()

    ctx = [conv(cin, cout) for _, _, cin, cout in CONTEXT_LAYERS]
    unet = []
    for name, kind, cin, cout in REFINE_LAYERS:
        if kind == "convT":
            unet.append(convT(cin, cout))
        else:
            unet.append(conv(cin, cout, REFINE_HEAD_SCALE if name == "out" else 1.0))
    return {"context": ctx, "unet": unet}
