"""Time the full transforms and their engine launches (diagnostics): phi = total - engine."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0910_5435_b200 as bb
from oracle import sht_oracle
l = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sht = bb.SHT(l)
beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, 1)).cuda()
grid = torch.empty((B, 2 * l, 4 * l - 1), dtype=torch.complex128, device="cuda")
out = torch.empty_like(beta)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {"syn": [], "ana": []}
for k in range(12):
    if k == 2:
        sht.engine_time(True)  # from here on: timed iterations only
    for name, fn in (("syn", lambda: sht.synthesize(beta, out=grid)), ("ana", lambda: sht.analyze(grid, out=out))):
        flush.fill_(k)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if k >= 2: res[name].append(a.elapsed_time(b) * 1e3)
ms, n = sht.engine_time(False)
eng = [1e3 * ms[d] / n[d] for d in range(2)]
syn = sum(res["syn"]) / len(res["syn"]); ana = sum(res["ana"]) / len(res["ana"])
print(f"l={l} B={B} synth {syn:.1f} us (engine {eng[0]:.1f}, phi {syn - eng[0]:.1f}) | analysis {ana:.1f} us (engine {eng[1]:.1f}, phi {ana - eng[1]:.1f})")
