import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1401_2720_b200 as J
from paper_1401_2720_b200 import _dev
n = 16384
t0=time.time(); x = torch.empty((n, n), dtype=torch.float64, pin_memory=True); print("pin alloc 2GB", time.time()-t0)
t0=time.time(); y = torch.empty((n, n), dtype=torch.float64); y.fill_(0); print("pageable alloc+touch 2GB", time.time()-t0)
d = torch.randn(n, n, dtype=torch.float64, device='cuda'); torch.cuda.synchronize()
t0=time.time(); h = d.cpu(); torch.cuda.synchronize(); print("D2H pageable 2GB", time.time()-t0)
t0=time.time(); x.copy_(d, non_blocking=True); torch.cuda.synchronize(); print("D2H pinned 2GB", time.time()-t0)
t0=time.time(); d2 = x.to('cuda', non_blocking=True); torch.cuda.synchronize(); print("H2D pinned 2GB", time.time()-t0)
t0=time.time(); _ = _dev._to_host(d); print("_to_host 2GB", time.time()-t0)
t0=time.time(); s = J.Solver(n, J.SolverConfig()); torch.cuda.synchronize(); print("Solver init", time.time()-t0)
t0=time.time(); s = J.Solver(n, J.SolverConfig()); torch.cuda.synchronize(); print("Solver init again", time.time()-t0)
t0=time.time(); ok = bool(torch.isfinite(d).all()); print("isfinite", time.time()-t0)
