"""Tightness of the piecewise-sum bound vs LB_Keogh at the final tau (oracle, CPU; analysis only).
usage: python scripts/paa_tightness.py [C5]"""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import datagen, oracle
from numpy.lib.stride_tricks import sliding_window_view as swv
c = datagen.CONFIGS[sys.argv[1] if len(sys.argv)>1 else "C5"]
NQ = 8
qs, _ = datagen.make(c, N=0)
qs = qs[:NQ]
db = datagen.series(c.family, c.N, c.n, c.seed, datagen.ROLE_DB, c.znorm, start=0)
t=time.time()
idx, dist, _ = oracle.nn_twopass(qs, db, c.w, c.p, c.k, threads=8)
print("oracle", time.time()-t)
tau = dist[:, -1].astype(np.float64) ** c.p
w=c.w; n=c.n
def env(y):
    yp = np.pad(y, (w, w), mode='edge')
    v = swv(yp, 2*w+1)
    return v.max(1), v.min(1)
dbd = db.astype(np.float64)
for qi in range(NQ):
    U, L = env(qs[qi].astype(np.float64))
    # LB_Keogh^p
    lbk = np.zeros(len(db))
    for s in range(0, len(db), 100000):
        x = dbd[s:s+100000]
        d = np.maximum(np.maximum(x - U, L - x), 0)
        lbk[s:s+100000] = (d**c.p).sum(1)
    out = [f"q{qi} tau={tau[qi]:.3f} keogh_surv={np.mean(lbk<=tau[qi]):.4f}"]
    for seg in (4, 8, 16, 32):
        S = n // seg
        xs = dbd.reshape(len(db), S, seg).sum(2)
        Us = U.reshape(S, seg).sum(1); Ls = L.reshape(S, seg).sum(1)
        d = np.maximum(np.maximum(xs - Us, Ls - xs), 0)
        b = (d**c.p).sum(1) / (seg if c.p == 2 else 1)
        assert np.all(b <= lbk * (1 + 1e-9) + 1e-9)
        out.append(f"seg{seg}:{np.mean(b<=tau[qi]):.4f}")
    print(" ".join(out), flush=True)
