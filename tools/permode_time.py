import sys, torch
sys.path.insert(0, '.')
import paper_2504_11681_b200 as T
from paper_2504_11681_b200.permode import prepare_weights, run_layer_permode
for case in [(128,128,128,512,512,64,64,2),(32,64,64,256,256,32,32,2),(1024,64,64,1,1024,1,128,1)]:
    cfg = T.FnoLayerConfig(*case)
    x = torch.randn(cfg.batch, cfg.hidden_dim, cfg.dim_x, cfg.dim_y, dtype=torch.complex64, device='cuda')
    w = torch.randn(cfg.hidden_dim, cfg.output_dim, cfg.keep_x, cfg.keep_y, dtype=torch.complex64, device='cuda')
    wp = prepare_weights(w)
    for _ in range(2): run_layer_permode(cfg, x, w_prepared=wp)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): y = run_layer_permode(cfg, x, w_prepared=wp)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    w2 = torch.randn(cfg.hidden_dim, cfg.output_dim, dtype=torch.complex64, device='cuda')
    for _ in range(2): T.run_layer_device(cfg, x, w2)
    torch.cuda.synchronize(); s.record()
    for _ in range(5): T.run_layer_device(cfg, x, w2)
    e.record(); torch.cuda.synchronize()
    print(case, 'permode ms', round(ms, 3), 'shared-W ms', round(s.elapsed_time(e) / 5, 3), flush=True)
    del x, y
    torch.cuda.empty_cache()
