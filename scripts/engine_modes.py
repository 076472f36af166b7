"""Engine time per direction under diagnostic modes (results are wrong for
modes != 0): 0 normal, 1 stream only (no records), 4 records + barriers
without panel arithmetic."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0910_5435_b200 as bb
from paper_0910_5435_b200._lib import lib, check
from oracle import sht_oracle
l = int(sys.argv[1]) if len(sys.argv) > 1 else 256
sht = bb.SHT(l)
beta = torch.from_numpy(sht_oracle.random_coefficients(l, 1, 1)).cuda()
grid = torch.empty((1, 2 * l, 4 * l - 1), dtype=torch.complex128, device="cuda")
out = torch.empty_like(beta)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in (0, 1, 4):
    check(lib().bfly_sht_debug(sht._h, mode))
    for k in range(10):
        if k == 2:
            sht.engine_time(True)
        flush.fill_(k)
        sht.synthesize(beta, out=grid)
        flush.fill_(k)
        sht.analyze(grid, out=out)
    torch.cuda.synchronize()
    ms, n = sht.engine_time(False)
    print(f"mode {mode}: engine synthesis {1e3 * ms[0] / n[0]:.1f} us, analysis {1e3 * ms[1] / n[1]:.1f} us")
