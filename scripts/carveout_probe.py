"""Diagnostics: engine launch time back to back vs. after a kernel that runs
with the default L1/shared-memory carveout (SM reconfiguration cost)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0910_5435_b200 as bb
l = int(sys.argv[1]) if len(sys.argv) > 1 else 32
plans = bb.build_glrow_planset(l, 1e-12)
ps = bb.PlanSet(plans)
x, nrhs = ps.stack([torch.zeros(1)] * 0) if False else (None, 4)
n_in = sum(p.n_cols for p in plans) * nrhs
n_out = sum(p.n_rows for p in plans) * nrhs
xin = torch.randn(n_in, dtype=torch.float64, device="cuda")
out = torch.empty(n_out, dtype=torch.float64, device="cuda")
other = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
def run(interleave):
    ts = []
    for k in range(30):
        if interleave:
            other.fill_(k)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); ps.apply_device(xin, out, nrhs); b.record()
        torch.cuda.synchronize()
        if k >= 5: ts.append(a.elapsed_time(b) * 1e3)
    return sum(ts) / len(ts)
print(f"l={l}: engine back to back {run(False):.1f} us, after a default-carveout kernel {run(True):.1f} us")
