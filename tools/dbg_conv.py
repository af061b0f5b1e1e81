import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2112_10603_b200.convtc import conv2d, pack_conv, cpad_of
for (cin, cout, s, H, W, nt) in [(16,16,2,256,448,16),(16,16,1,128,224,16),(16,16,1,128,224,32),(32,32,1,64,112,32),(64,64,1,32,56,64),(16,16,1,128,256,16),(16, 32, 1, 64, 64, 32)]:
    x = torch.randn(2, H, W, cpad_of(cin), device='cuda').to(torch.bfloat16)
    w = torch.randn(cout, cin, 3, 3, device='cuda')
    b = torch.zeros(cout, device='cuda')
    try:
        y = conv2d(x, pack_conv(w, cpad_of(cin), nt), b, cout, 3, s, 1, ntile=nt)
        torch.cuda.synchronize()
        ref = torch.relu(torch.nn.functional.conv2d(x.float().permute(0,3,1,2)[:, :cin], w, b, stride=s, padding=1)).permute(0,2,3,1)
        print(cin, cout, s, H, W, nt, "ok", (y[..., :cout].float() - ref).abs().max().item())
    except Exception as e:
        print(cin, cout, s, H, W, nt, "FAIL", e)
