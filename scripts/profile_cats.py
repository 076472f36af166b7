"""Per-category consumer-warp cycle breakdown of one engine launch (diagnostics)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0910_5435_b200 as bb
from paper_0910_5435_b200._lib import lib, check
from oracle import sht_oracle
l = int(sys.argv[1]) if len(sys.argv) > 1 else 256
sht = bb.SHT(l)
n = sht.info()["n_jobs"]
beta = torch.from_numpy(sht_oracle.random_coefficients(l, 1, 1)).cuda()
gb = torch.empty(sht.phi_shape(1), dtype=torch.complex128, device="cuda")
names = ["wait_stage", "barrier", "loadz", "sel", "tpanel", "spanel", "pro/epilogue", "total"]
check(lib().bfly_sht_debug(sht._h, 2))
for direction in ("synthesis", "analysis"):
    check(lib().bfly_sht_trace(sht._h, max(n, 8)))
    if direction == "synthesis":
        sht.legendre_synthesize(beta, out=gb)
    else:
        sht.legendre_analyze(gb, out=torch.empty_like(beta))
    torch.cuda.synchronize()
    buf = np.zeros((max(n, 8), 4), np.uint64)
    check(lib().bfly_sht_trace_read(sht._h, buf.ctypes.data_as(C.c_void_p), max(n, 8)))
    v = buf.reshape(-1)[:8].astype(float)
    cnt = buf.reshape(-1)[8:16].astype(float)
    tot = v[7]
    print(direction, " ".join("%s %.1f%%" % (nm, 100 * x / tot) for nm, x in zip(names[:7], v[:7])),
          "| accounted %.1f%%" % (100 * v[:7].sum() / tot))
    print("   cycles per event (per warp):", " ".join("%s %.0f" % (nm, x / max(c, 1)) for nm, x, c in zip(names[:7], v[:7], cnt[:7])),
          "| warps", int(cnt[7]), "cycles/warp %.0f" % (tot / max(cnt[7], 1)))
