"""Engine build variants at a batched configuration (diagnostics).

usage: python scripts/batch_variants.py LIB[,LIB...] [L] [B]
Builds (or reloads from /tmp) the device program once with the default
library, then for each library variant times the full transform pair and the
engine launches alone (CUDA events, L2 flushed before each step)."""
import json
import os
import subprocess
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_0910_5435_b200 as bb
from oracle import sht_oracle
l, B, cache = int(os.environ["L"]), int(os.environ["B"]), os.environ["CACHE"]
if os.path.exists(cache):
    sht = bb.SHT.load(cache)
else:
    sht = bb.SHT(l, eps=1e-12)
    sht.save(cache)
beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=5, decaying_member=B - 1)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
grid = sht.synthesize(beta); back = sht.analyze(grid)
err = (torch.linalg.vector_norm(back - beta) / torch.linalg.vector_norm(beta)).item()
sht.engine_time(True)
ts = []
for k in range(6):
    flush.fill_(k)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); g = sht.synthesize(beta); sht.analyze(g, out=back); b.record(); torch.cuda.synchronize()
    if k >= 2: ts.append(a.elapsed_time(b))
ms, n = sht.engine_time(False)
step = sum(ts) / len(ts)
print(json.dumps({"step_ms": round(step, 3), "pairs_s": round(B / step * 1e3, 1),
                  "engine_ms": [round(m / max(c, 1), 3) for m, c in zip(ms, n)], "rt": err,
                  "smem": sht.info()["smem_bytes"]}))
'''


def main():
    libs = sys.argv[1].split(",")
    l = sys.argv[2] if len(sys.argv) > 2 else "1024"
    B = sys.argv[3] if len(sys.argv) > 3 else "16"
    cache = f"/tmp/bfly_prog_l{l}.bin"
    for lib in libs:
        env = dict(os.environ, ROOT=root, L=l, B=B, CACHE=cache)
        if lib != "default":
            env["BFLY_LIB"] = os.path.join(root, lib)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        print(lib, p.stdout.strip() or p.stderr.strip()[-400:], flush=True)


if __name__ == "__main__":
    main()
