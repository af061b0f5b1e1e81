"""tcgen05 implicit-GEMM convolution vs torch (fp32 math on the same bf16 operands)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    return torch


def _nhwc(torch, x, cpad):
    B, C, H, W = x.shape
    out = torch.zeros((B, H, W, cpad), dtype=torch.bfloat16, device=x.device)
    out[..., :C] = x.permute(0, 2, 3, 1).to(torch.bfloat16)
    return out


def _check(torch, got_nhwc, ref_nchw, cout, out_f32):
    got = got_nhwc[..., :cout].permute(0, 3, 1, 2).float()
    ref = ref_nchw if out_f32 else ref_nchw.to(torch.bfloat16).float()
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    # fp32 accumulation in a different order + one bf16 rounding of the output
    assert err <= (1e-4 if out_f32 else 1.6e-2) * scale, (err, scale)


@pytest.mark.parametrize("cin,cout,k,s,H,W,relu,out_f32", [
    (6, 128, 3, 2, 36, 70, True, False),       # VIBlock conv0 shape class (cpad 16, SW32)
    (17, 128, 3, 2, 40, 132, True, False),     # 17 input channels (cpad 32, SW64)
    (128, 256, 3, 2, 20, 66, True, False),     # conv1 (cpad 128, SW128, N = 256)
    (256, 256, 3, 1, 10, 260, True, False),    # residual 256x256, two pixel tiles per row
    (64, 16, 3, 1, 9, 17, False, True),        # fp32 output, N = 16 tile
    (128, 20, 3, 1, 13, 150, False, True),     # N = 32 tile, SW128: row-reuse tiles (4 rows, ragged H)
    (128, 32, 3, 1, 6, 40, True, False),       # row-reuse, bf16 output
    # row-reuse tiles for every small-N class RefineNet uses (ntile 16/32/64 x SW 32/64/128)
    (16, 3, 3, 1, 37, 200, False, True),       # the RefineNet head: 16 -> 3, fp32 out, NT16 / SW32
    (16, 16, 3, 1, 19, 130, True, False),      # ContextNet x1: NT16 / SW32
    (32, 32, 3, 1, 23, 70, True, False),       # U-Net d0b: NT32 / SW64
    (64, 64, 3, 1, 11, 300, True, False),      # U-Net d1b: NT64 / SW128
    (32, 16, 3, 1, 9, 129, True, False),       # NT16 / SW64
    (128, 16, 3, 1, 5, 40, False, False),      # NT16 / SW128
    (16, 32, 3, 1, 14, 33, True, False),       # NT32 / SW32
    (32, 64, 3, 1, 7, 150, True, False),       # NT64 / SW64
])
def test_conv_matches_torch(torch_cuda, cin, cout, k, s, H, W, relu, out_f32):
    torch = torch_cuda
    from paper_2112_10603_b200 import convtc
    g = torch.Generator(device="cuda").manual_seed(cin * 1000 + cout)
    x = torch.randn((2, cin, H, W), device="cuda", generator=g)
    w = torch.randn((cout, cin, k, k), device="cuda", generator=g) / (cin * k * k) ** 0.5
    b = torch.randn((cout,), device="cuda", generator=g) * 0.1
    xb, wb = x.to(torch.bfloat16).float(), w.to(torch.bfloat16).float()
    ref = torch.nn.functional.conv2d(xb, wb, b, stride=s, padding=1)
    if relu:
        ref = torch.relu(ref)
    cpad = convtc.cpad_of(cin)
    nt = convtc.ntile_of(cout)
    got = convtc.conv2d(_nhwc(torch, x, cpad), convtc.pack_conv(w, cpad, nt), b.float().contiguous(), cout,
                        k, s, 1, relu=relu, out_f32=out_f32)
    torch.cuda.synchronize()
    _check(torch, got, ref, cout, out_f32)


@pytest.mark.parametrize("cin,cout,H,W,relu,out_f32", [
    (256, 128, 9, 30, True, False),
    (128, 5, 17, 33, False, True),             # the 5-channel flow/mask head
])
def test_convT_matches_torch(torch_cuda, cin, cout, H, W, relu, out_f32):
    torch = torch_cuda
    from paper_2112_10603_b200 import convtc
    g = torch.Generator(device="cuda").manual_seed(cin + cout)
    x = torch.randn((2, cin, H, W), device="cuda", generator=g)
    w = torch.randn((cin, cout, 4, 4), device="cuda", generator=g) / (cin * 4) ** 0.5
    b = torch.randn((cout,), device="cuda", generator=g) * 0.1
    xb, wb = x.to(torch.bfloat16).float(), w.to(torch.bfloat16).float()
    ref = torch.nn.functional.conv_transpose2d(xb, wb, b, stride=2, padding=1)
    if relu:
        ref = torch.relu(ref)
    cpad = convtc.cpad_of(cin)
    nt = convtc.ntile_of(cout)
    got = convtc.conv2d(_nhwc(torch, x, cpad), convtc.pack_convT(w, cpad, nt), b.float().contiguous(), cout,
                        4, 2, 1, transposed=True, relu=relu, out_f32=out_f32)
    torch.cuda.synchronize()
    _check(torch, got, ref, cout, out_f32)


@pytest.mark.parametrize("cin,cout,H,W,relu,out_f32", [
    (64, 16, 17, 150, True, False),    # RefineNet u3: 64 -> 16, N = 64 (row-reuse tiles)
    (128, 32, 9, 60, True, False),     # RefineNet u2: N = 128
    (128, 5, 13, 40, False, True),     # the VINet head shape, fp32
])
def test_convT_subpixel_matches_torch(torch_cuda, cin, cout, H, W, relu, out_f32):
    """ConvTranspose2d(k4 s2 p1) as one 3x3 sub-pixel GEMM (fvv_conv_desc.transposed = 2)."""
    torch = torch_cuda
    from paper_2112_10603_b200 import convtc
    g = torch.Generator(device="cuda").manual_seed(cin * 7 + cout)
    x = torch.randn((2, cin, H, W), device="cuda", generator=g)
    w = torch.randn((cin, cout, 4, 4), device="cuda", generator=g) / (cin * 4) ** 0.5
    b = torch.randn((cout,), device="cuda", generator=g) * 0.1
    xb, wb = x.to(torch.bfloat16).float(), w.to(torch.bfloat16).float()
    ref = torch.nn.functional.conv_transpose2d(xb, wb, b, stride=2, padding=1)
    if relu:
        ref = torch.relu(ref)
    cpad = convtc.cpad_of(cin)
    nt = convtc.ntile_of(4 * cout)
    got = convtc.conv2d(_nhwc(torch, x, cpad), convtc.pack_convT_subpixel(w, cpad, nt), b.float().repeat(4).contiguous(),
                        cout, 4, 2, 1, transposed=True, subpixel=True, relu=relu, out_f32=out_f32)
    torch.cuda.synchronize()
    _check(torch, got, ref, cout, out_f32)
