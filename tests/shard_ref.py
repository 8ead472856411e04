"""Host reference of nn_merge for the sharded-protocol tests (test-only code)."""
import torch


def merge_reference(g_idx: torch.Tensor, g_dst: torch.Tensor):
    """k smallest by (dist, idx) of the G*k entries per query, ignoring idx < 0 (padding)."""
    G, Q, k = g_idx.shape
    out_i = torch.full((Q, k), -1, dtype=torch.int64)
    out_d = torch.full((Q, k), float("inf"), dtype=torch.float32)
    for q in range(Q):
        cand = [(float(g_dst[g, q, j]), int(g_idx[g, q, j])) for g in range(G) for j in range(k)
                if int(g_idx[g, q, j]) >= 0]
        cand.sort()
        for r, (d, i) in enumerate(cand[:k]):
            out_i[q, r] = i
            out_d[q, r] = d
    return out_i, out_d
