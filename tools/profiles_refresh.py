"""Summarise a gpurun evidence batch into profiles/ (run here, no GPU).

Inputs in gpurun_out/: bench_default.json, bench_ref.json, launches.csv (ncu
launch list), fine_full.ncu-rep (ncu --set full of one fine launch).

  python tools/profiles_refresh.py <tag>      # e.g. r1c
"""

import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
UPDATES = 256 * 1024 * 128 * 500
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x"]


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main(tag):
    # bench lines
    json.dump({"default_bench_line": last_json(os.path.join(OUT, "bench_default.json")),
               "reference_arm_line": last_json(os.path.join(OUT, "bench_ref.json"))},
              open(os.path.join(PROF, f"{tag}_bench_lines.json"), "w"), indent=1)
    # launch list
    rows = [r for r in csv.reader(open(os.path.join(OUT, "launches.csv"))) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    fine = []
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[r[ki]][0] += 1
        agg[r[ki]][1] += v
        if "fine_kernel" in r[ki]:
            fine.append(v / 1e6)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(PROF, f"{tag}_launch_list.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none --csv:\n"
                "#   python bench.py --steps 2 --warmup 3 --no-cpu --no-extras\n"
                "# cold-cache, serialised per-launch times: compare SHARES (bench.py's CUDA events\n"
                "# give the absolute numbers); field_kernel launches are input setup outside the\n"
                "# timed region; fine launches = 3 warm-up + 2 timed + 2 pipeline warm-up + 2 e2e\n")
        f.write("launches  total_ms  share  kernel\n")
        for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{n:8d} {v / 1e6:9.3f} {100 * v / tot:6.2f}%  {k}\n")
        f.write("\n# per-launch fine_kernel times (ms): " + ", ".join(f"{x:.3f}" for x in fine) + "\n")
    # ncu full capture
    rep = os.path.join(OUT, "fine_full.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    H, U, V = rr[0], rr[1], rr[2]
    get = lambda k: V[H.index(k)]  # noqa: E731
    rd, wr = float(get("dram__bytes_read.sum")) * 1e9, float(get("dram__bytes_write.sum")) * 1e9
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    tmp = os.path.join(OUT, "_src.csv")
    open(tmp, "w").write(src)
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "25"],
                           capture_output=True, text=True).stdout
    with open(os.path.join(PROF, f"{tag}_fine_kernel_ncu.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on -k regex:fine_kernel -c 1\n"
                "#   python bench.py --steps 1 --warmup 3 --no-cpu --no-extras "
                "(cfg5: 256 x 1024x128, 500 steps)\n")
        f.write(f"# kernel: {get('Kernel Name')}\n\n")
        for k in KEYS:
            if k in H:
                f.write(f"{k:75s} {U[H.index(k)]:10s} {V[H.index(k)]}\n")
        f.write(f"\n# algorithmic bytes per launch: {UPDATES * 16 / 1e9:.1f} GB; measured DRAM "
                f"{(rd + wr) / 1e9:.1f} GB ({(rd + wr) / UPDATES:.2f} B/update)\n")
        f.write("\n# warp-stall samples by source line (tools/ncu_lines.py)\n" + lines)
    json.dump({"source": f"ncu --set full, gpurun_out/fine_full.ncu-rep ({tag})",
               "kernel": get("Kernel Name"), "nx": 1024, "nv": 128, "instances": 256, "steps": 500,
               "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
               "bytes_per_launch": int(rd + wr), "bytes_per_update": round((rd + wr) / UPDATES, 3),
               "algorithmic_bytes_per_update": 16,
               "gpu_time_ms_cold": float(get("gpu__time_duration.sum"))},
              open(os.path.join(PROF, "fine_kernel_traffic.json"), "w"), indent=1)
    print("wrote", tag)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "latest")
