import torch, sys
sys.path.insert(0, '.')
import paper_2412_08832_b200 as hc
elems = 1 << 28
xs = {dt: torch.randn(elems, device='cuda').to(dt) for dt in (torch.float16, torch.bfloat16)}
q = torch.empty(elems, dtype=torch.uint8, device='cuda')
for n in (16384, 32768):
    sc = torch.empty(elems // n, device='cuda')
    def L(dt):
        hc.hadacore_fwht_quant(xs[dt].view(-1, n), 'e4m3', out=q.view(torch.float8_e4m3fn).view(-1, n), row_scale=sc)
    for pattern in ('same16', 'same16', 'alt', 'alt', 'same_bf', 'pairs'):
        seq = {'same16': [torch.float16]*10, 'alt': [torch.float16, torch.bfloat16]*5, 'same_bf': [torch.bfloat16]*10,
               'pairs': [torch.float16, torch.float16, torch.bfloat16, torch.bfloat16]*3}[pattern]
        L(seq[0]); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for dt in seq: L(dt)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / len(seq)
        print(n, pattern, f"{(3 * elems + 4 * elems / n) / (ms * 1e-3) / 1e9:.1f} GB/s  {ms*1e3:.1f} us/launch")
