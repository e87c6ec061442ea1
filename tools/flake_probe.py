import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import test_determinism as td
td.REPS = 6
for trial in range(int(os.environ.get("TRIALS", "1"))):
    outs = td._ensemble_run(256, 128, 256, 12, 0)
    ref = outs[0]
    bad = False
    for r, o in enumerate(outs[1:], 1):
        for name, a, b in zip(("rho", "E", "g"), o[:3], ref[:3]):
            if not np.array_equal(a, b):
                bad = True
                d = np.argwhere(a != b)
                print(f"trial {trial} rep {r} {name}: {len(d)} differing entries; slices {sorted(set(d[:,0]))[:10]}, rows {sorted(set(d[:,1]))[:20] if d.shape[1]>1 else ''}, cols {sorted(set(d[:,2]))[:16] if d.shape[1]>2 else ''}; layout {o[3]}")
                i = tuple(d[0]); print("   first:", i, a[i], b[i], "is b NaN/zero?", np.isnan(b[i]), b[i]==0)
    print("trial", trial, "layout", ref[3], "bad" if bad else "ok")
