"""Engine configuration sweep (diagnostics): kernel time per direction for
build variants (consumer warps / CTAs per SM) x stage capacities."""
import os, subprocess, sys, json
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_0910_5435_b200 as bb
from oracle import sht_oracle
l = int(os.environ.get("L", "256"))
sht = bb.SHT(l)
beta = torch.from_numpy(sht_oracle.random_coefficients(l, 1, 1)).cuda()
gb = torch.empty(sht.phi_shape(1), dtype=torch.complex128, device="cuda")
out = torch.empty_like(beta)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, fn in (("syn", lambda: sht.legendre_synthesize(beta, out=gb)), ("ana", lambda: sht.legendre_analyze(gb, out=out))):
    ts = []
    for k in range(8):
        flush.fill_(k)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if k >= 3: ts.append(a.elapsed_time(b) * 1e3)
    res[name] = round(sum(ts) / len(ts), 1)
res["smem"] = sht.info()["smem_bytes"]
print(json.dumps(res))
'''
for lib in sys.argv[1].split(","):
    for kb in sys.argv[2].split(","):
        env = dict(os.environ, ROOT=root, BFLY_LIB=os.path.join(root, lib), BFLY_STAGE_KB=kb)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        print(lib, kb, p.stdout.strip() or p.stderr.strip()[-300:], flush=True)
