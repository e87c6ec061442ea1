import os, sys, time
sys.path.insert(0, "/root/repo") if os.path.isdir("/root/repo") else None
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2511_13386_b200 as pk
import paper_2511_13386_b200.parareal as ppl
from paper_2511_13386_b200 import configs
c = configs.cfg4(); m = c.mesh
th = pk.Thresholds(1e-3, 1e-3)
cfg_full = pk.PararealConfig(eps=c.eps, t_final=2.0, ng=64, k_max=1, tol=1e-8, thresholds=th, options=pk.HybridOptions(adaptation=True))
E0 = pk.solve_field(c.rho, c.rho_bar, m, rtol=1e-5)
fluid_p, kin_p = ppl.default_params(cfg_full, m, E0)
fs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
t_red = 64 * fs * kin_p.dt
cfg = pk.PararealConfig(eps=c.eps, t_final=t_red, ng=64, k_max=1, tol=1e-8, thresholds=th, options=pk.HybridOptions(adaptation=True))
eng = ppl._Engine(cfg, m, c.rho, c.g, c.rho_bar, fluid_p, kin_p)
eng.coarse_sweep()
for name, X, wins in (("rows1-8", eng.row[1:9].clone(), list(range(2, 10))),
                      ("rho0x8", eng.row[0:1].repeat(8, 1).clone(), list(range(2, 10)))):
    for cnt_on in (False, True):
        cnt = torch.zeros((8, 2), dtype=torch.int64, device=X.device)
        eng.be.fine(X, wins); torch.cuda.synchronize()
        if cnt_on: eng.be.dev.count_rows(cnt)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); eng.be.fine(X, wins); e1.record(); torch.cuda.synchronize()
        eng.be.dev.count_rows(None)
        print(name, "count" if cnt_on else "plain", f"{e0.elapsed_time(e1)/fs*1e3:.1f} us/step", eng.be.dev.last_launch(), cnt.sum(0).tolist())
