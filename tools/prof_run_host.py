import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_2511_13386_b200 as pk
from paper_2511_13386_b200 import configs, parareal
c = configs.cfg2()
cfg = pk.PararealConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10, options=pk.HybridOptions(adaptation=False))
for _ in range(3):
    torch.cuda.synchronize(); t0=time.perf_counter()
    res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
    torch.cuda.synchronize(); print("wall %.2f ms"%((time.perf_counter()-t0)*1e3), res.iterations)
pr = cProfile.Profile(); pr.enable()
res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(35)
