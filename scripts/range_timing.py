"""Legendre-stage timing of an order range (SHT.range) for B functions:
python scripts/range_timing.py L MU0 MU1 B  -> JSON (ms per direction, TF/s)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402

l, mu0, mu1, B = (int(x) for x in sys.argv[1:5])
os.environ.setdefault("BFLY_WAVES", "1")
sht = bb.SHT.range(l, mu0, mu1, eps=1e-12)
N = 4 * l - 1
dev = torch.device("cuda", 0)
beta = torch.randn((B, 4 * l * l), dtype=torch.complex128, device=dev)
g = torch.zeros((N, B, 2 * l), dtype=torch.complex128, device=dev)
b = torch.zeros_like(beta)
for _ in range(2):
    sht.legendre_synthesize(beta, out=g)
    sht.legendre_analyze(g, out=b)
torch.cuda.synchronize()
sht.engine_time(True)
K = 5
for _ in range(K):
    sht.legendre_synthesize(beta, out=g)
    sht.legendre_analyze(g, out=b)
torch.cuda.synchronize()
ms, n = sht.engine_time(False)
W = sht.info()["stored_words"]
fl = 2 * 4 * B * W
out = {"l": l, "mu": [mu0, mu1], "B": B, "ms": [ms[0] / K, ms[1] / K],
       "tflops": [fl / (ms[0] / K * 1e-3) / 1e12, fl / (ms[1] / K * 1e-3) / 1e12], "lib": os.environ.get("BFLY_LIB", "")}
print(json.dumps(out))
