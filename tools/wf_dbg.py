import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2504_11681_b200 as T
from oracle import fnofuse_port as O
for shape in [(3, 16, 16, 1, 256, 1, 32, 1), (2, 8, 8, 1, 1024, 1, 128, 1)]:
    cfg = T.FnoLayerConfig(*shape)
    print(shape, T.layer_schedule(cfg, "fully_fused"), flush=True)
    x, w = O.random_inputs(cfg, 1)
    y = T.run_layer_device(cfg, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    print("err", T.max_rel_error(y.cpu().numpy(), O.run_layer_values(cfg, x, w)), flush=True)
