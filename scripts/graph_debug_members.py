"""Per-member agreement of the wave-program (graph) transforms with the
whole-chain engine (one function per call) and the round trip."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import sht_oracle  # noqa: E402

l, B = int(sys.argv[1]), int(sys.argv[2])
beta = torch.from_numpy(sht_oracle.random_coefficients(l, B, seed=6500 + l, decaying_member=B - 1)).cuda()
os.environ["BFLY_WAVES"] = "1"
wv = bb.SHT(l, eps=1e-12)
os.environ["BFLY_WAVES"] = "0"
eng = bb.SHT(l, eps=1e-12)
rel = lambda x, y: float(torch.linalg.vector_norm(x - y) / torch.linalg.vector_norm(y))  # noqa: E731
g = wv.synthesize(beta)
g0 = torch.cat([eng.synthesize(beta[i:i + 1]) for i in range(B)])
print("synth vs engine per member", ["%.1e" % rel(g[i], g0[i]) for i in range(B)])
b = wv.analyze(g0)
b0 = torch.cat([eng.analyze(g0[i:i + 1]) for i in range(B)])
print("anal vs engine per member", ["%.1e" % rel(b[i], b0[i]) for i in range(B)])
print("round trip per member", ["%.1e" % rel(wv.analyze(g)[i], beta[i]) for i in range(B)])
