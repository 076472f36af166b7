"""One synthesis + analysis of l = L, B functions on the wave programs (for
ncu captures of the graph kernel): python scripts/graph_once.py L B"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import sht_oracle  # noqa: E402

l, B = int(sys.argv[1]), int(sys.argv[2])
os.environ.setdefault("BFLY_WAVES", "1")
sht = bb.SHT(l, eps=1e-12)
beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=5)).cuda()
for _ in range(2):
    g = sht.synthesize(beta)
    b = sht.analyze(g)
torch.cuda.synchronize()
print("round trip", float((torch.linalg.vector_norm(b - beta) / torch.linalg.vector_norm(beta)).item()))
