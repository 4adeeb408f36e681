"""Summarise the ncu --set full captures of tools/profile_round.sh into
profiles/<round>_ncu_full_summary.json (+ <round>_traffic.json, the bench's
roofline.traffic source).  Algorithmic bytes per launch follow SURVEY.md
8(d) for the C3 hierarchy (256^3 dam-break) level shapes."""
import csv
import io
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
N0, Z0 = 16777216, 117047296   # level 0
N1, Z1 = 8347648, 91350080     # level 1
N2, Z2 = 2605983, 38621109     # level 2
ALG = {  # name: (key, algorithmic bytes per launch, formula)
    # level 0 runs in symmetric-stencil form (k_dia): diagonal +
    # 3 upper diagonals + a 1-byte row mask = 33 bytes per row
    "smooth_L0": ("vcycle_smooth@0", 33 * N0 + 32 * N0, "33*n + 32*n (D + 3 upper diagonals + mask; x, f, w, out)"),
    "down_L0": ("vcycle_down@0", 33 * N0 + 24 * N0, "33*n + 24*n (symmetric-stencil form; u0 folded: w replaces u0)"),
    "down_L1": ("vcycle_down@1", 10 * Z1 + 4 * (N1 + 1) + 24 * N1, "10*nnz + 4*(n+1) + 24*n (2-byte column codes)"),
    # k_rap_grp (round 2): the Galerkin product + the fine level's fused damped-Jacobi rebuild
    "rap_L0": ("rap@0", 12 * Z0 + 8 * Z1 + 4 * N0 + 4 * (N1 + 1) + 20 * N0,
               "12*nnz_f + 8*nnz_c + 4*n_f + 4*(n_c+1) + 20*n_f (fused Jacobi)"),
    "rap_L1": ("rap@1", 12 * Z1 + 8 * Z2 + 4 * N1 + 4 * (N2 + 1) + 20 * N1,
               "12*nnz_f + 8*nnz_c + 4*n_f + 4*(n_c+1) + 20*n_f (fused Jacobi)"),
}
WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2]


summary, traffic = {}, {}
for name, (key, alg, formula) in ALG.items():
    rep = os.path.join("gpurun_out", name + ".ncu-rep")
    if not os.path.exists(rep):
        continue
    hdr, units, vals = raw(rep)
    d = {w: f"{vals[hdr.index(w)]} {units[hdr.index(w)]}".strip() for w in WANT if w in hdr}
    rd = float(vals[hdr.index("dram__bytes_read.sum")]) * UNIT[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(vals[hdr.index("dram__bytes_write.sum")]) * UNIT[units[hdr.index("dram__bytes_write.sum")]]
    t_us = float(vals[hdr.index("gpu__time_duration.sum")])
    d.update({"dram_total_GB": round((rd + wr) / 1e9, 4), "algorithmic_GB": round(alg / 1e9, 4),
              "algorithmic_formula": formula, "traffic_over_algorithmic": round((rd + wr) / alg, 3),
              "algorithmic_GB_s_at_ncu_time": round(alg / t_us / 1e3, 1),
              "note": "ncu replays each kernel with cold caches and serialised launches; time is not the bench value"})
    summary[key] = d
    traffic[key] = rd + wr
json.dump(summary, open(os.path.join(OUT, f"{R}_ncu_full_summary.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(OUT, f"{R}_traffic.json"), "w"), indent=1)
print(json.dumps({k: (v["dram_total_GB"], v["algorithmic_GB"], v["gpu__time_duration.sum"]) for k, v in summary.items()}))
