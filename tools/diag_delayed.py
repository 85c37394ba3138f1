import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from test_gpu_delayed import *
for lr in (1e-3, 3e-4):
  for S in (1, 3):
    for T in (5,):
        depth,w,dims=18,8,(40,48,40)
        desc = rn.net_desc(depth, w, dims)
        genes, unit_stage = contiguous_genes(desc, S) if S > 1 else (None, [0]*len(O.Net(depth,w,dims).units))
        net = O.Net(depth, w, dims)
        arrays = synthetic.perturb_params(net.tensors, synthetic.init_params(net.tensors, seed=0))
        flat = np.concatenate([a.ravel() for a in arrays]).astype(np.float32)
        bs = [synthetic.make_batch(2, *dims, seed=10 + t) for t in range(T)]
        res = run_delayed(desc, 2, rn.RN_F32, S, genes, flat, bs, lr)
        ref = O.delayed_pipeline_train(net, arrays, bs, lr, unit_stage)
        w_gpu = merged_weights(res, net.tensors, unit_stage)
        delta = ref["params"] - flat.astype(np.float64)
        sgd = O.delayed_pipeline_train(net, arrays, bs, lr, [0]*len(net.units))
        print(lr, S, T, np.linalg.norm(sgd['params']-ref['params'])/np.linalg.norm(delta), np.linalg.norm(w_gpu.astype(np.float64) - ref["params"]) / np.linalg.norm(delta), max(abs(np.array(res[0]["losses"])-ref["losses"])/np.array(ref["losses"])))
