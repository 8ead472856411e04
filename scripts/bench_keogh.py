"""Time the LB_Keogh tile kernel alone (dense C-ABI lb_keogh) on C5-like shapes.
Usage: DTWLB_KEOGH_VAR=<v> python scripts/bench_keogh.py [Q] [N] [n] [p]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_0811_3301_b200 import lb_envelope, lb_keogh

Q, N, n, p = (int(a) for a in (sys.argv[1:5] + ["2048", "1000000", "256", "2"][len(sys.argv[1:5]):]))
qs = torch.from_numpy(datagen.random_walks(Q, n, seed=1, role=1)).cuda()
db = torch.from_numpy(datagen.random_walks(N, n, seed=2)).cuda()
U, L = lb_envelope(qs, 25)
env = torch.stack([U, L]).contiguous()
out = lb_keogh(env, db, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 3
for _ in range(reps):
    out = lb_keogh(env, db, p)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
el = Q * N * n
print(f"var={os.environ.get('DTWLB_KEOGH_VAR', '0')} Q={Q} N={N} n={n} p={p}: {ms:.2f} ms  "
      f"{el / ms / 1e9:.2f} Telem/s  {el / ms / 1e9 / (148 * 1.965):.2f} elem/clk/SM")
