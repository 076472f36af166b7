"""Check every interpolative decomposition of GPU-built plans against the dense
matrix: python scripts/gpubuild_debug.py L EPS [MU0 MU1] [--host]
Replays the depth-first build in numpy (which source columns every stripe
holds) and reports, per ID, the residual ||B[:, others] - B[:, sel] T||_F /
(eps_used ||B||_F) and max |T|.  Test tooling (uses the oracle for the dense matrix)."""
import os
import struct
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5435_b200 as bb  # noqa: E402
from oracle import ref  # noqa: E402


def parse(blob):
    pos = 5
    assert blob[:5] == b"BFLY1"

    def u64():
        nonlocal pos
        v = struct.unpack_from("<Q", blob, pos)[0]
        pos += 8
        return v

    def f64():
        nonlocal pos
        v = struct.unpack_from("<d", blob, pos)[0]
        pos += 8
        return v

    def mat(r, c):
        nonlocal pos
        m = np.frombuffer(blob, dtype="<f8", count=r * c, offset=pos).reshape(c, r).T
        pos += 8 * r * c
        return m

    p = {"n_rows": u64(), "n_cols": u64(), "eps": f64(), "width": u64(), "levels": u64(), "events": [], "roots": []}
    for _ in range(u64()):
        kind = blob[pos]
        pos += 1
        ev = {"kind": kind, "ids": []}
        if kind == 0:
            ev["c0"], ev["nc"] = u64(), u64()
        elif kind == 1:
            ev["left"] = [u64() for _ in range(u64())]
        for _ in range(u64()):
            rank, others = u64(), u64()
            sel = [u64() for _ in range(rank)]
            ev["ids"].append((sel, mat(rank, others)))
        p["events"].append(ev)
    for _ in range(u64()):
        g = []
        for _ in range(u64()):
            rb, rc, rank = u64(), u64(), u64()
            g.append((rb, rc, mat(rc, rank)))
        p["roots"].append(g)
    return p


def spans(l, level):
    part = [(0, l)]
    for _ in range(level - 1):
        nxt = []
        for b, c in part:
            t = (c + 1) // 2
            nxt += [(b, t), (b + t, c - t)]
        part = nxt
    return part


def np_id(blk, e):
    """The kernel's algorithm in numpy: pivoted Householder QR with exact trailing norms."""
    w = np.array(blk, dtype=float, order="F")
    m, n = w.shape
    fro = np.linalg.norm(w)
    thr = e * fro / np.sqrt(n)
    perm = np.arange(n)
    k = 0
    for j in range(min(m, n)):
        nr = (w[j:, j:] ** 2).sum(axis=0)
        p = j + int(np.argmax(nr))
        if j > 0 and np.sqrt(nr[p - j]) <= thr:
            break
        if p != j:
            w[:, [j, p]] = w[:, [p, j]]
            perm[[j, p]] = perm[[p, j]]
        x = w[j:, j].copy()
        sigma = np.linalg.norm(x)
        alpha = -sigma if x[0] >= 0 else sigma
        v = x.copy()
        v[0] -= alpha
        vn2 = v @ v
        if vn2 > 0:
            w[j:, j + 1:] -= np.outer(v, (2.0 / vn2) * (v @ w[j:, j + 1:]))
        w[j:, j] = 0.0
        w[j, j] = alpha
        k = j + 1
    t = np.linalg.solve(w[:k, :k], w[:k, k:]) if k < n else np.zeros((k, 0))
    return perm[:k], perm[k:], t


def check(plan, a, eps, tag):
    l = a.shape[0]
    cn = np.linalg.norm(a, axis=0)
    stack = []
    worst = 0.0
    for ei, ev in enumerate(plan["events"]):
        if ev["kind"] == 0:
            cols = np.arange(ev["c0"], ev["c0"] + ev["nc"])
            ins = [((0, l), cols, -1.0)]
            lv = 1
        else:
            top = stack.pop()
            lv = top[0] + 1
            if ev["kind"] == 1:
                left = stack.pop()
                cats = [np.concatenate([x, y]) for x, y in zip(left[1], top[1])]
            else:
                cats = top[1]
            part = spans(l, lv)
            ins = []
            for s, cat in enumerate(cats):
                nn = float(np.sqrt((cn[cat] ** 2).sum()))
                for h in range(2):
                    ins.append((part[2 * s + h], cat, nn))
        assert len(ins) == len(ev["ids"]), (tag, ei, len(ins), len(ev["ids"]))
        out = []
        for ii, (((r0, m), cols, nn), (sel, t)) in enumerate(zip(ins, ev["ids"])):
            blk = a[r0:r0 + m][:, cols]
            fro = np.linalg.norm(blk)
            e = eps if nn < 0 or fro == 0 else min(0.5, max(eps, eps * nn / fro))
            sel = np.asarray(sel, dtype=int)
            oth = np.setdiff1d(np.arange(len(cols)), sel)
            res = np.linalg.norm(blk[:, oth] - blk[:, sel] @ t) if len(oth) else 0.0
            q = res / (e * fro) if fro > 0 else 0.0
            tm = float(np.abs(t).max()) if t.size else 0.0
            if q > 3.0 or tm > 2.5:
                print(f"  BAD {tag} event {ei} kind {ev['kind']} id {ii}: rows [{r0},{r0 + m}) n={len(cols)} rank={len(sel)} "
                      f"res/(eps fro)={q:.3e} eps_used={e:.2e} fro={fro:.3e} max|T|={tm:.3f}")
                if len(oth):
                    best = np.linalg.lstsq(blk[:, sel], blk[:, oth], rcond=None)[0]
                    rb = np.linalg.norm(blk[:, oth] - blk[:, sel] @ best) / (e * fro)
                    s2, o2, t2 = np_id(blk, e)
                    r2 = np.linalg.norm(blk[:, o2] - blk[:, s2] @ t2) / (e * fro)
                    print(f"      best T for this skeleton: {rb:.3e}; |T - best|max {np.abs(t - best).max():.3e}; numpy mirror: rank "
                          f"{len(s2)} res {r2:.3e}; same skeleton set: {set(s2.tolist()) == set(sel.tolist())}; "
                          f"same pivot order: {s2.tolist() == sel.tolist()}")
            worst = max(worst, q)
            out.append(cols[sel])
        stack.append((lv, out))
    # roots
    assert len(stack) == len(plan["roots"]), (tag, len(stack), len(plan["roots"]))
    for (lv, outs), g in zip(stack, plan["roots"]):
        part = spans(l, lv)
        for (r0, m), src, (rb, rc, s) in zip(part, outs, g):
            assert (rb, rc) == (r0, m), (tag, rb, rc, r0, m)
            d = np.abs(s - a[r0:r0 + m][:, src]).max() if s.size else 0.0
            if d > 1e-10 * max(1e-300, np.abs(s).max() if s.size else 0.0):
                print(f"  BAD {tag} root rows [{r0},{r0 + m}): skeleton differs from the source columns by {d:.3e}")
    return worst


def main():
    l = int(sys.argv[1])
    eps = float(sys.argv[2])
    args = [x for x in sys.argv[3:] if not x.startswith("--")]
    mu0, mu1 = (int(args[0]), int(args[1])) if len(args) >= 2 else (0, 2 * l)
    os.environ["BFLY_BUILDER"] = "host" if "--host" in sys.argv else "gpu"
    os.environ.setdefault("BFLY_BUILD_VERBOSE", "1")
    nodes, rho, _ = ref.rule(0, l, 0)
    plans = bb.build_glrow_planset(l, eps, mu_range=(mu0, mu1), rule=(nodes, rho))
    print("built", len(plans), "plans", flush=True)
    if "--twice" in sys.argv:
        again = bb.build_glrow_planset(l, eps, mu_range=(mu0, mu1), rule=(nodes, rho))
        diff = [i for i, (x, y) in enumerate(zip(plans, again)) if x.to_bfly1() != y.to_bfly1()]
        print("second build: plans with different bytes:", len(diff), diff[:16], flush=True)
    keys = [(mu, p) for mu in range(mu0, mu1) for p in (0, 1) if bb.chain_cols(l, mu, p) > 0]
    worst = 0.0
    step = max(1, len(keys) // int(os.environ.get("DEBUG_SAMPLE", "64")))
    for i in range(0, len(keys), step):
        mu, p = keys[i]
        a = ref.dense_glrow(l, mu, p)
        w = check(parse(plans[i].to_bfly1()), a, eps, f"(mu={mu}, p={p})")
        worst = max(worst, w)
    print("worst residual / (eps fro):", worst)


if __name__ == "__main__":
    main()
