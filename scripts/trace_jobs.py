"""Per-job timeline of one engine launch (diagnostics; prints a summary)."""
import sys, os, ctypes as C, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0910_5435_b200 as bb
from paper_0910_5435_b200._lib import lib, check
from oracle import sht_oracle
l = int(sys.argv[1]) if len(sys.argv) > 1 else 256
sht = bb.SHT(l)
if len(sys.argv) > 2:
    check(lib().bfly_sht_debug(sht._h, int(sys.argv[2])))
info = sht.info()
n = info["n_jobs"]
beta = torch.from_numpy(sht_oracle.random_coefficients(l, 1, 1)).cuda()
gb = torch.empty(sht.phi_shape(1), dtype=torch.complex128, device="cuda")
out = {}
for direction in ("synthesis", "analysis"):
    for rep in range(3):
        check(lib().bfly_sht_trace(sht._h, n))
        if direction == "synthesis":
            sht.legendre_synthesize(beta, out=gb)
        else:
            sht.legendre_analyze(gb, out=torch.empty_like(beta))
        torch.cuda.synchronize()
    buf = np.zeros((n, 4), np.uint64)
    check(lib().bfly_sht_trace_read(sht._h, buf.ctypes.data_as(C.c_void_p), n))
    t0 = buf[:, 0].min()
    st = (buf[:, 0] - t0) / 1e3
    en = (buf[:, 1] - t0) / 1e3
    dur = en - st
    order = np.argsort(-dur)
    print(direction, "kernel span us %.1f" % en.max(), "first start %.2f" % st.min(), "last start %.2f" % st.max())
    print("  longest jobs (task, start, dur us, stages):", [(int(i), round(float(st[i]), 1), round(float(dur[i]), 1), int(buf[i, 3])) for i in order[:8]])
    print("  dur percentiles 50/90/99:", np.percentile(dur, [50, 90, 99]).round(2), "mean", dur.mean().round(2))
    print("  stage rate (stages/us) for biggest jobs:", [round(float(buf[i, 3] / dur[i]), 2) for i in order[:5]])
    out[direction] = {"span": float(en.max()), "dur": dur.tolist(), "stages": buf[:, 3].tolist(), "start": st.tolist()}
json.dump(out, open(os.path.join("gpurun_out", f"trace_l{l}.json"), "w"))
