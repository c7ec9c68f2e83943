"""Helpers shared by the -m gpu tests: run the CUDA path through the C ABI binding."""
import numpy as np
import torch

import paper_2210_15114_b200 as l1


def gpu_matvec(X, Z, k_begin=0, k_end=None, ws_limit=None, host=False, mode="auto"):
    """Prepare X and run one query through the C ABI.  X, Z: numpy or torch (any device).
    mode: the query strategy ("auto" | "gather" | "scatter", include/l1dm.h)."""
    Xt = torch.as_tensor(np.ascontiguousarray(X)) if isinstance(X, np.ndarray) else X
    Zt = torch.as_tensor(np.ascontiguousarray(Z)) if isinstance(Z, np.ndarray) else Z
    if host:
        h = l1.l1dm_prepare(Xt.cpu(), k_begin, k_end)
    else:
        h = l1.l1dm_prepare(Xt.cuda(), k_begin, k_end)
    if ws_limit is not None:
        l1.l1dm_set_workspace_limit(h, ws_limit)
    l1.l1dm_set_query_mode(h, mode)
    if host:
        Y = l1.l1dm_matvec(h, Zt.cpu())
    else:
        Y = l1.l1dm_matvec(h, Zt.cuda())
        torch.cuda.synchronize()
    l1.l1dm_sync(h)
    out = Y.cpu().numpy()
    l1.l1dm_free(h)
    return out
