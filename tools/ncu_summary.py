"""Summarise one `ncu --set full` report into a profiles/ text file (run here,
no GPU): the headline metrics of the first profiled launch, DRAM bytes
against an optional algorithmic byte count, and the warp-stall samples by
source line (tools/ncu_lines.py).

  python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r2_x_ncu.txt "title" [alg_bytes]
"""

import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "sm__cycles_elapsed.avg.per_second"]


def main(rep, out, title, alg=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    H, U, V = rr[0], rr[1], rr[2]
    get = lambda k: V[H.index(k)]  # noqa: E731
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    tmp = os.path.join(ROOT, "gpurun_out", "_src.csv")
    open(tmp, "w").write(src)
    lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "25"],
                           capture_output=True, text=True).stdout
    with open(out, "w") as f:
        f.write(f"# {title}\n# kernel: {get('Kernel Name')}\n# report: {os.path.basename(rep)} "
                f"({len(rr) - 2} profiled launch(es); first shown)\n\n")
        if len(rr) > 3:
            f.write("# all profiled launches: kernel | duration | registers | issue active % | "
                    "FP64 pipe % | DRAM bytes r+w\n")
            for row in rr[2:]:
                g = lambda k: row[H.index(k)] if k in H else "-"  # noqa: E731
                f.write(f"#   {g('Kernel Name')[:60]:60s} | {g('gpu__time_duration.sum')} "
                        f"{U[H.index('gpu__time_duration.sum')]} | {g('launch__registers_per_thread')}"
                        f" | {g('smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
                        f"{g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')} | "
                        f"{g('dram__bytes_read.sum')}+{g('dram__bytes_write.sum')}\n")
            f.write("\n")
        for k in KEYS:
            if k in H:
                f.write(f"{k:75s} {U[H.index(k)]:12s} {V[H.index(k)]}\n")
        rd = float(get("dram__bytes_read.sum").replace(",", "")) if "dram__bytes_read.sum" in H else 0
        wr = float(get("dram__bytes_write.sum").replace(",", "")) if "dram__bytes_write.sum" in H else 0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(U[H.index("dram__bytes_read.sum")], 1)
        wr *= scale.get(U[H.index("dram__bytes_write.sum")], 1)
        f.write(f"\n# DRAM bytes (read + write): {(rd + wr) / 1e6:.3f} MB")
        if alg:
            f.write(f"; algorithmic {float(alg) / 1e6:.3f} MB ({(rd + wr) / float(alg):.2f}x)")
        f.write("\n\n# warp-stall samples by source line (tools/ncu_lines.py)\n" + lines)
    print("wrote", out)


if __name__ == "__main__":
    main(*sys.argv[1:])
