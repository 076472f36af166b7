"""Real-field SHT pair timing (RC = 2 engine + shared-DFT phi) vs the complex pair."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0910_5435_b200 as bb
l = int(sys.argv[1]) if len(sys.argv) > 1 else 256
sht = bb.SHT(l)
rng = np.random.default_rng(1)
n = l * (2 * l + 1)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
half = torch.from_numpy(rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))).cuda()
full = torch.from_numpy(bb.full_from_half(l, half.cpu().numpy())).cuda()
grid_r = torch.empty((B, 2 * l, 4 * l - 1), dtype=torch.float64, device="cuda")
back_r = torch.empty_like(half)
grid_c = torch.empty((B, 2 * l, 4 * l - 1), dtype=torch.complex128, device="cuda")
back_c = torch.empty_like(full)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(fn, K=30):
    ev = []
    for k in range(K + 5):
        flush.fill_(k)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        if k >= 5: ev.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3
t_real = run(lambda: (sht.synthesize_real(half, out=grid_r), sht.analyze_real(grid_r, out=back_r)))
t_cplx = run(lambda: (sht.synthesize(full, out=grid_c), sht.analyze(grid_c, out=back_c)))
print(f"l={l} B={B}: real fields {B * 1e6 / t_real:.0f} pairs/s, complex {B * 1e6 / t_cplx:.0f} pairs/s")
