"""Diagnostics (run under ncu): one engine synthesis launch per debug mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0910_5435_b200 as bb
from paper_0910_5435_b200._lib import lib, check
from oracle import sht_oracle
sht = bb.SHT(256)
beta = torch.from_numpy(sht_oracle.random_coefficients(256, 1, 1)).cuda()
gb = torch.empty(sht.phi_shape(1), dtype=torch.complex128, device="cuda")
for mode in (0, 1, 4):
    check(lib().bfly_sht_debug(sht._h, mode))
    for k in range(3):
        sht.legendre_synthesize(beta, out=gb)
    torch.cuda.synchronize()
