"""fp32 torch reference of VINet -- the oracle of the north-star CNN path.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's CPU
legs).  The reference package has no CNN; SURVEY.md sec. 8(c)
prescribes this oracle: a torch fp32 module written from PAPER.md:100-126,
320-337 with seeded random weights (paper_2112_10603_b200/vinet_params.py).
Every operation is spelled out (no grid_sample / interpolate) so the CUDA
engine restates the same arithmetic:

  pool2(x)     2x2 mean ((a + b) + (c + d)) * 0.25            image pyramid
  up2(x)       2x bilinear, align_corners=False: grid ((i + 0.5) / 2 - 0.5),
               clamped, x-lerp then y-lerp                     flow / mask
  warp(I, F)   backward bilinear at (x + fx, y + fy), clamped to the plane,
               i0 = min(floor(s), n - 2), out = (1-ay)((1-ax)a + ax b) + ay((1-ax)c + ax d)
  canvas       the network runs on the image edge-padded (replicate, bottom/right) to
               multiples of 64 (three 2x pools + four stride-2 layers); the flows
               are cropped back to H x W before synthesis
  synth        m = sigmoid(M); for view t: F_l,t = 2t F_l, F_r,t = 2(1-t) F_r,
               w_t = (1-t) m / ((1-t) m + t (1-m)); out = w_t warp(I_l) + (1-w_t) warp(I_r)
               per plane (chroma: flow = 2x2 mean * 0.5, mask = 2x2 mean), rint, clip.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as Fn

GRAY8, YUV420, RGB8 = 0, 1, 2


def planes_of(frame: np.ndarray, w: int, h: int, fmt: int):
    """Packed frame bytes -> list of uint8 planes (H, W[, 3])."""
    if fmt == GRAY8:
        return [frame[:w * h].reshape(h, w)]
    if fmt == RGB8:
        return [frame[:w * h * 3].reshape(h, w, 3)]
    cw, ch = (w + 1) // 2, (h + 1) // 2
    y = frame[:w * h].reshape(h, w)
    u = frame[w * h:w * h + cw * ch].reshape(ch, cw)
    v = frame[w * h + cw * ch:w * h + 2 * cw * ch].reshape(ch, cw)
    return [y, u, v]


def net_image(frame: np.ndarray, w: int, h: int, fmt: int) -> torch.Tensor:
    """(3, H, W) float32 in [0, 1] (vinet_params docstring)."""
    p = planes_of(frame, w, h, fmt)
    if fmt == RGB8:
        x = torch.from_numpy(p[0].astype(np.float32)).permute(2, 0, 1)
    elif fmt == YUV420:
        u = np.repeat(np.repeat(p[1], 2, 0), 2, 1)[:h, :w]
        v = np.repeat(np.repeat(p[2], 2, 0), 2, 1)[:h, :w]
        x = torch.from_numpy(np.stack([p[0], u, v]).astype(np.float32))
    else:
        y = p[0].astype(np.float32)
        x = torch.from_numpy(np.stack([y, np.full_like(y, 127.5), np.full_like(y, 127.5)]))
    return x * (1.0 / 255.0)


def pool2(x: torch.Tensor) -> torch.Tensor:
    a, b = x[..., 0::2, 0::2], x[..., 0::2, 1::2]
    c, d = x[..., 1::2, 0::2], x[..., 1::2, 1::2]
    return ((a + b) + (c + d)) * 0.25


def _taps(n_out: int, n_in: int, device=None):
    s = (torch.arange(n_out, dtype=torch.float32, device=device) + 0.5) * 0.5 - 0.5
    s = s.clamp(0.0, float(n_in - 1))
    i0 = torch.clamp(torch.floor(s), max=max(n_in - 2, 0)).long()
    i1 = torch.clamp(i0 + 1, max=n_in - 1)
    return i0, i1, s - i0.float()


def up2(x: torch.Tensor) -> torch.Tensor:
    """(..., h, w) -> (..., 2h, 2w) bilinear, align_corners=False."""
    h, w = x.shape[-2:]
    y0, y1, fy = _taps(2 * h, h, x.device)
    x0, x1, fx = _taps(2 * w, w, x.device)
    top = x[..., y0, :]
    bot = x[..., y1, :]
    rows = (1.0 - fy)[:, None] * top + fy[:, None] * bot
    left, right = rows[..., x0], rows[..., x1]
    return (1.0 - fx) * left + fx * right


def warp(img: torch.Tensor, fx: torch.Tensor, fy: torch.Tensor) -> torch.Tensor:
    """img (..., H, W), flow (H, W): backward bilinear with clamped coordinates."""
    H, W = img.shape[-2:]
    ys = torch.arange(H, dtype=torch.float32, device=img.device)[:, None]
    xs = torch.arange(W, dtype=torch.float32, device=img.device)[None, :]
    sx = (xs + fx).clamp(0.0, float(W - 1))
    sy = (ys + fy).clamp(0.0, float(H - 1))
    x0 = torch.clamp(torch.floor(sx), max=W - 2).long()
    y0 = torch.clamp(torch.floor(sy), max=H - 2).long()
    ax, ay = sx - x0.float(), sy - y0.float()
    flat = img.reshape(*img.shape[:-2], H * W)

    def at(yy, xx):
        return flat[..., (yy * W + xx).reshape(-1)].reshape(*img.shape[:-2], H, W)

    a, b = at(y0, x0), at(y0, x0 + 1)
    c, d = at(y0 + 1, x0), at(y0 + 1, x0 + 1)
    top = (1.0 - ax) * a + ax * b
    bot = (1.0 - ax) * c + ax * d
    return (1.0 - ay) * top + ay * bot


def block_forward(x: torch.Tensor, layers) -> torch.Tensor:
    """One VIBlock on (1, cin, h, w) -> (1, 5, h, w)."""
    (w0, b0), (w1, b1) = layers[0], layers[1]
    y = torch.relu(Fn.conv2d(x, w0, b0, stride=2, padding=1))
    y = torch.relu(Fn.conv2d(y, w1, b1, stride=2, padding=1))
    for k in range(2, 8):
        w, b = layers[k]
        y = torch.relu(Fn.conv2d(y, w, b, stride=1, padding=1))
    w, b = layers[8]
    y = torch.relu(Fn.conv_transpose2d(y, w, b, stride=2, padding=1))
    w, b = layers[9]
    return Fn.conv_transpose2d(y, w, b, stride=2, padding=1)


def canvas(w: int, h: int):
    return (w + 63) // 64 * 64, (h + 63) // 64 * 64


def pad_canvas(x: torch.Tensor, w: int, h: int) -> torch.Tensor:
    wp, hp = canvas(w, h)
    ys = torch.clamp(torch.arange(hp, device=x.device), max=h - 1)
    xs = torch.clamp(torch.arange(wp, device=x.device), max=w - 1)
    return x[..., ys, :][..., xs]


@torch.no_grad()
def flows(left: np.ndarray, right: np.ndarray, w: int, h: int, fmt: int, params, device=None):
    """VINet on one pair -> (5, H, W) float32: F_l (2), F_r (2), mask logit (1) at full resolution.
    device: where the fp32 oracle runs (CPU by default; a CUDA device only speeds the checker up,
    with TF32 disabled by the caller)."""
    if device is not None:
        params = [[(w_.to(device), b_.to(device)) for w_, b_ in blk] for blk in params]
    il = [pad_canvas(net_image(left, w, h, fmt).to(device or "cpu"), w, h)]
    ir = [pad_canvas(net_image(right, w, h, fmt).to(device or "cpu"), w, h)]
    for _ in range(2):
        il.insert(0, pool2(il[0]))
        ir.insert(0, pool2(ir[0]))
    state = None
    for i in range(3):
        a, b = il[i], ir[i]
        if state is None:
            x = torch.cat([a, b], 0)
        else:
            st = up2(state)
            st[0:4] = st[0:4] * 2.0
            wl = warp(a, st[0], st[1])
            wr = warp(b, st[2], st[3])
            x = torch.cat([a, b, wl, wr, st], 0)
            state = st
        res = block_forward(x[None], params[i])[0]
        state = res if state is None else state + res
    return state[:, :h, :w].contiguous().cpu()


def _synth_plane(pl: torch.Tensor, pr: torch.Tensor, fl, fr, wgt, t: float) -> torch.Tensor:
    a = warp(pl, fl[0] * (2.0 * t), fl[1] * (2.0 * t))
    b = warp(pr, fr[0] * (2.0 * (1.0 - t)), fr[1] * (2.0 * (1.0 - t)))
    v = wgt * a + (1.0 - wgt) * b
    return torch.clamp(torch.round(v), 0.0, 255.0)  # torch.round: half to even


@torch.no_grad()
def synth(left: np.ndarray, right: np.ndarray, w: int, h: int, fmt: int, state: torch.Tensor, t: float):
    """Direct-t view at t in (0, 1) from the VINet state -> packed uint8 frame."""
    m = torch.sigmoid(state[4])
    wt = (1.0 - t) * m / ((1.0 - t) * m + t * (1.0 - m))
    pls, prs = planes_of(left, w, h, fmt), planes_of(right, w, h, fmt)
    out = []
    if fmt == RGB8:
        pl = torch.from_numpy(pls[0].astype(np.float32)).permute(2, 0, 1)
        pr = torch.from_numpy(prs[0].astype(np.float32)).permute(2, 0, 1)
        out.append(_synth_plane(pl, pr, state[0:2], state[2:4], wt, t).permute(1, 2, 0))
    else:
        out.append(_synth_plane(torch.from_numpy(pls[0].astype(np.float32)),
                                torch.from_numpy(prs[0].astype(np.float32)), state[0:2], state[2:4], wt, t))
        if fmt == YUV420:
            fc = pool2(state[0:4]) * 0.5
            wc = pool2(wt)
            for k in (1, 2):
                out.append(_synth_plane(torch.from_numpy(pls[k].astype(np.float32)),
                                        torch.from_numpy(prs[k].astype(np.float32)), fc[0:2], fc[2:4], wc, t))
    return np.concatenate([o.numpy().astype(np.uint8).reshape(-1) for o in out])


# ---------------------------------------------------------------------------
# RefineNet + ContextNet (vinet_params.CONTEXT_LAYERS / REFINE_LAYERS)
# ---------------------------------------------------------------------------
def _conv(x, wb, stride):
    w, b = wb
    return torch.relu(Fn.conv2d(x, w, b, stride=stride, padding=1))


def contextnet(img: torch.Tensor, flow: torch.Tensor, layers):
    """img (3, Hp, Wp) canvas image, flow (2, Hp, Wp) canvas flow -> 4 warped feature maps."""
    f = img[None]
    feats = []
    for k in range(4):
        f = _conv(f, layers[2 * k], 2)
        f = _conv(f, layers[2 * k + 1], 1)
        flow = pool2(flow) * 0.5
        feats.append(warp(f[0], flow[0], flow[1]))
    return feats


def refine_inputs(left, right, w: int, h: int, fmt: int, state: torch.Tensor, t: float):
    """(x0 (17, Hp, Wp) canvas U-Net input, merged (3, H, W), F_l,t, F_r,t canvas flows)."""
    a, b = net_image(left, w, h, fmt), net_image(right, w, h, fmt)
    fl, fr = state[0:2] * (2.0 * t), state[2:4] * (2.0 * (1.0 - t))
    m = torch.sigmoid(state[4])
    wt = (1.0 - t) * m / ((1.0 - t) * m + t * (1.0 - m))
    wl = warp(a, fl[0], fl[1])
    wr = warp(b, fr[0], fr[1])
    merged = wt * wl + (1.0 - wt) * wr
    x0 = torch.cat([a, b, wl, wr, wt[None], fl, fr], 0)
    return pad_canvas(x0, w, h), merged, pad_canvas(fl, w, h), pad_canvas(fr, w, h)


@torch.no_grad()
def refine_view(left, right, w: int, h: int, fmt: int, state: torch.Tensor, t: float, rparams):
    """Direct-t view at t refined by RefineNet -> (packed uint8 frame, refined (3, H, W) f32 in [0, 1])."""
    x0, merged, fl, fr = refine_inputs(left, right, w, h, fmt, state, t)
    il = pad_canvas(net_image(left, w, h, fmt), w, h)
    ir = pad_canvas(net_image(right, w, h, fmt), w, h)
    cl = contextnet(il, fl, rparams["context"])
    cr = contextnet(ir, fr, rparams["context"])
    u = rparams["unet"]
    s0 = _conv(_conv(x0[None], u[0], 2), u[1], 1)
    s1 = _conv(_conv(torch.cat([s0, cl[0][None], cr[0][None]], 1), u[2], 2), u[3], 1)
    s2 = _conv(_conv(torch.cat([s1, cl[1][None], cr[1][None]], 1), u[4], 2), u[5], 1)
    s3 = _conv(_conv(torch.cat([s2, cl[2][None], cr[2][None]], 1), u[6], 2), u[7], 1)

    def up(x, wb):
        return torch.relu(Fn.conv_transpose2d(x, wb[0], wb[1], stride=2, padding=1))
    x = up(torch.cat([s3, cl[3][None], cr[3][None]], 1), u[8])
    x = up(torch.cat([x, s2], 1), u[9])
    x = up(torch.cat([x, s1], 1), u[10])
    x = up(torch.cat([x, s0], 1), u[11])
    r = torch.sigmoid(Fn.conv2d(x, u[12][0], u[12][1], padding=1))[0, :, :h, :w]
    out = torch.clamp(merged + (r * 2.0 - 1.0), 0.0, 1.0)
    return pack_image(out, w, h, fmt), out


def pack_image(img: torch.Tensor, w: int, h: int, fmt: int) -> np.ndarray:
    """(3, H, W) in [0, 1] -> packed uint8 frame: RGB interleaved, Y (+ 2x2-mean U, V), or Y."""
    v = img * 255.0
    if fmt == RGB8:
        return torch.clamp(torch.round(v), 0, 255).permute(1, 2, 0).numpy().astype(np.uint8).reshape(-1)
    y = torch.clamp(torch.round(v[0]), 0, 255).numpy().astype(np.uint8).reshape(-1)
    if fmt == GRAY8:
        return y
    c = torch.clamp(torch.round(pool2(v[1:3])), 0, 255).numpy().astype(np.uint8)
    return np.concatenate([y, c[0].reshape(-1), c[1].reshape(-1)])
