import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from test_gpu_multirank import *
for Mb in (1, 2):
    dims = (40, 48, 40)
    desc = rn.net_desc(18, 64, dims)
    loads = rn.net_units(desc)[2]
    genes = rn.gabra_place_slack(loads, 2, seed=7, require_all_used=1)[0]
    tensors = rn.net_params(desc)[0]
    arrays = synthetic.perturb_params(tensors, synthetic.init_params(tensors, seed=0))
    flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
    x, y = synthetic.make_batch(4, *dims, seed=1)
    hyb = run_ranks(4, lambda r: step_rank(desc, 2, rn.RN_BF16, r, 4, 2, genes, Mb, rn.local_transport_id(), flat, x, y) if False else None) if False else None
    nid = rn.local_transport_id()
    hyb = run_ranks(4, lambda r: step_rank(desc, 2, rn.RN_BF16, r, 4, 2, genes, Mb, nid, flat, x, y))
    nid2 = rn.local_transport_id()
    dp = run_ranks(2, lambda r: step_rank(desc, 2, rn.RN_BF16, r, 2, 1, None, Mb, nid2, flat, x, y))
    masks = [owner_mask(tensors, desc, genes, 2, s) for s in range(2)]
    g_h = np.where(masks[0], hyb[0]["g"], hyb[1]["g"])
    print("Mb", Mb, "genes", genes, "loss", hyb[0]["loss"], dp[0]["loss"])
    off = 0
    for name, shape, _ in tensors:
        n = int(np.prod(shape))
        a, b = g_h[off:off+n], dp[0]["g"][off:off+n]
        if not np.array_equal(a, b):
            print("  differs", name, rel(a, b))
        off += n
