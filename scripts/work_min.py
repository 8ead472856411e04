"""Work of the survivor passes vs their order-independent minimum (GPU, analysis only).

For a sample of queries of a config: the final tau (from nn_search), the dense gate
bound (piecewise sums), LB_Keogh and LB_Improved over the whole database, and the
counts #{bound <= tau_final (1+eps)} -- the minimum number of evaluations any
processing order must do -- next to the counts at tau_1, the k-th best DTW of the S
lowest-gate candidates (what range 2 sees after a range-1 walk of size S).
usage: python scripts/work_min.py [C5] [nq]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import datagen  # noqa: E402
from paper_0811_3301_b200 import dtw_band, lb_envelope, lb_improved, lb_keogh, lb_piecewise, nn_search  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
NQ = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c = datagen.CONFIGS[name]
t = time.time()
qs, db = datagen.make(c)
print(f"datagen {time.time() - t:.1f}s", flush=True)
dev = torch.device("cuda")
q_t = torch.from_numpy(qs).to(dev)
db_t = torch.from_numpy(db).to(dev)
idx, dist = nn_search(q_t, db_t, c.w, c.p, c.k)
torch.cuda.synchronize()
sel = torch.linspace(0, c.Q - 1, NQ).long().to(dev)
qsub = q_t[sel].contiguous()
tau = dist[sel, -1].double() ** c.p * (1 + 1e-3)
U, L = lb_envelope(qsub, c.w)
env = torch.stack([U, L]).contiguous()
N = c.N
cnt = {}
for b in range(0, NQ, 32):
    e = env[:, b:b + 32].contiguous()
    qq = qsub[b:b + 32]
    tq = tau[b:b + 32, None]
    g = lb_piecewise(e, db_t, c.p).double() ** c.p
    k1 = lb_keogh(e, db_t, c.p).double() ** c.p
    k2 = lb_improved(qq, e, db_t, c.w, c.p).double() ** c.p
    for S in (2048, 8192, 32768, 131072):
        # tau_1 = k-th best DTW among the S lowest-gate candidates of each query
        gs, order = torch.topk(g, S, dim=1, largest=False)
        taus = []
        for r in range(qq.shape[0]):
            cand = order[r]
            d = dtw_band(db_t[cand].contiguous(), qq[r].expand(S, -1).contiguous(), c.w, c.p).double() ** c.p
            taus.append(torch.topk(d, c.k, largest=False).values[-1] * (1 + 1e-3))
        t1 = torch.stack(taus)[:, None]
        for nm, v in (("gate", g), ("keogh", k1), ("improved", k2)):
            cnt[(S, nm)] = cnt.get((S, nm), 0) + (v <= t1).sum().item()
    for nm, v in (("gate", g), ("keogh", k1), ("improved", k2)):
        cnt[("final", nm)] = cnt.get(("final", nm), 0) + (v <= tq).sum().item()
    print(f"block {b} done", flush=True)
tot = NQ * N
print(f"{name}: {NQ} queries x {N}; fraction of pairs with bound <= threshold")
for key in ["final", 2048, 8192, 32768, 131072]:
    print(f"  tau={key!s:>7}: gate {cnt[(key, 'gate')] / tot:.4f}  keogh {cnt[(key, 'keogh')] / tot:.4f}  "
          f"improved {cnt[(key, 'improved')] / tot:.4f}")
