"""Per-iteration timings of the cfg2 parareal run with and without the
overlapped correction/fine schedule."""
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2511_13386_b200 as pk
    from paper_2511_13386_b200 import configs, parareal

    c = configs.cfg2()
    cfg = pk.PararealConfig(eps=1e-2, t_final=0.5, ng=16, k_max=5, tol=1e-10,
                            options=pk.HybridOptions(adaptation=False))
    parareal.TIMELINE = True
    for ov in (False, True, False, True):
        parareal.OVERLAP = ov
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pk.run(cfg, c.rho, c.g, c.mesh, c.rho_bar)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tm = res.ledger.timings
        print(f"overlap={ov}: wall {wall * 1e3:.1f} ms, coarse {tm.coarse_sweep * 1e3:.1f}, "
              f"iterations {res.iterations}")
        ov = getattr(parareal, "_Overlap", None)
        for o in (ov._cache.values() if ov else []):
            print("   last iteration host enqueue %.2f ms" % (getattr(o, "host_enqueue_s", 0) * 1e3))
            print("   sweep enqueue %.2f ms, until swept %.2f ms" % (
                getattr(o, "sweep_enqueue_s", 0) * 1e3, getattr(o, "sweep_wait_s", 0) * 1e3))
            for n, fs, cr in getattr(o, "sweep_timeline", []):
                print(f"      sweep window {n:2d}: row ready {cr:7.2f} ms, its F starts {fs:7.2f} ms")
            for n, fs, fe, cr in getattr(o, "timeline", []):
                print(f"      window {n:2d}: F {fs:7.2f} .. {fe:7.2f} ms, corrected at {cr:7.2f} ms")
        for it in tm.iterations:
            print(f"   k={it['k']}: wall {it['wall_s'] * 1e3:.2f} ms, fine {it['parallel_s'] * 1e3:.2f}, "
                  f"corr {it['correction_s'] * 1e3:.2f}")


if __name__ == "__main__":
    main()
