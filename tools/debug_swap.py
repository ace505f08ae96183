import os, sys, traceback
os.environ["CUDA_LAUNCH_BLOCKING"] = "1"
sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2508_09591_b200 as hm
from paper_2508_09591_b200 import swap as S, traffic as T
wb = np.zeros((5, 4), bool)
for t, s in enumerate([{0}, {1}, {0, 2}, {0, 2}, {1, 3}]): wb[t, list(s)] = True
topo = hm.build_topology([2], 4, 1, 1)
params = hm.LevelParams((), (), (0.0,), (1.0,))
steps = [
 ("model", lambda: T._Model(wb, topo, params, None, True).fetch().times),
 ("partials", lambda: S._Partials(hm.device_mask(wb), 2).z.cpu()),
 ("tensors", lambda: hm.swap_tensors_incremental(wb, topo).intra),
 ("cost", lambda: hm.cost_matrix(hm.swap_tensors_incremental(wb, topo), topo, params, 1, 10.0)),
 ("smooth", lambda: hm.smooth_max([1.0, 2.0, 3.0], 10.0)),
 ("select", lambda: hm.select_swap(wb, topo, params, 10.0)),
]
for name, fn in steps:
    try:
        r = fn(); torch.cuda.synchronize(); print(name, "OK", r if not hasattr(r, "shape") else tuple(r.shape))
    except Exception as e:
        print(name, "FAIL", repr(e)[:300]); break
