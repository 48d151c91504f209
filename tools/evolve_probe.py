import time, numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2102_01732_b200 import SparseMLP, SGD
from synth import get_config
from synth.data import c5_host_rows
cfg = get_config("C5")
m = SparseMLP(cfg.sizes, cfg.epsilon, cfg.activation, cfg.alpha, cfg.dropout, cfg.init, cfg.model_seed, 0, cfg.batch)
B = cfg.batch
Xh, Yh = c5_host_rows(cfg, np.arange(2 * B))
xp = torch.from_numpy(Xh).pin_memory(); yp = torch.from_numpy(Yh.astype(np.int32)).pin_memory()
sgd = SGD(cfg.lr, cfg.momentum, cfg.weight_decay)
def ev(tag, e):
    torch.cuda.synchronize(); t0 = time.perf_counter(); m.evolve_topology(cfg.zeta, e); torch.cuda.synchronize()
    print(tag, round(time.perf_counter() - t0, 4), flush=True)
ev("first evolve (cold)", 0)
ev("second evolve", 1)
xd = torch.from_numpy(Xh[:B]).cuda(); yd = torch.from_numpy(Yh[:B].astype(np.int32)).cuda()
for s in range(3):
    m.forward(xd, train=True, step=s); m.backward(yd, fused=sgd)
ev("after device steps", 2)
for s in range(3):
    m.train_step_host(xp[:B], yp[:B], B, s, sgd)
ev("after sync host steps", 3)
lossp = torch.zeros(4).pin_memory()
for s in range(3):
    m.train_step_host_async(xp[:B], yp[:B], B, s, sgd, lossp[s:])
m.sync()
ev("after async host steps", 4)
ev("again", 5)
