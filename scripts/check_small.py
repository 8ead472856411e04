import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, datagen, oracle
from paper_0811_3301_b200 import nn_search
Q, N, k, p = (int(a) for a in sys.argv[1:5])
qs, db = datagen.make("C1", Q=Q, N=N)
try:
    idx, dist = nn_search(torch.from_numpy(qs).cuda(), torch.from_numpy(db).cuda(), 12, p, k)
    oi, od = oracle.nn_brute(qs, db, 12, p, k)
    print("Q N k p", Q, N, k, p, "ok" if np.array_equal(idx.cpu().numpy(), oi) else "MISMATCH")
except Exception as e:
    print("Q N k p", Q, N, k, p, "ERR", str(e)[:120])
