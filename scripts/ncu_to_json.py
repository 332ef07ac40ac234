"""Summarise an `ncu --set full` capture of k_solve into profiles/k_solve_ncu.json
(read by bench.py's roofline `traffic` / ncu fields when its source sha matches
the current library build) and a text summary.

usage: python scripts/ncu_to_json.py REP.ncu-rep SCENARIOS SUMMARY.txt "source description"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

STALLS = ["barrier", "long_scoreboard", "no_instruction", "selected", "short_scoreboard", "wait"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "s": 1.0, "ms": 1e-3, "us": 1e-6,
             "ns": 1e-9}

    def get(name):
        i = h.index(name)
        return float(vals[i].replace(",", "")) * scale.get(units[i], 1.0)
    return get


def main():
    rep, scenarios, summary, source = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
    g = raw(rep)
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    d = {
        "source": source,
        "library_source_sha256_16": bench.library_sha(),
        "scenarios": scenarios,
        "duration_s": g("gpu__time_duration.sum"),
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_solve": (rd + wr) / scenarios,
        "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_per_sm": g("sm__warps_active.avg.per_cycle_active"),
        "registers_per_thread": int(g("launch__registers_per_thread")),
        "shared_bank_conflicts_per_wavefront": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")
        / max(g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"), 1.0),
        "stalls_per_issue": {s: g(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio") for s in STALLS},
    }
    with open(os.path.join(ROOT, "profiles", "k_solve_ncu.json"), "w") as fh:
        json.dump(d, fh, indent=1)
    with open(summary, "w") as fh:
        fh.write(f"# ncu --set full of k_solve ({scenarios} cfg4 scenarios, one launch), source sha "
                 f"{d['library_source_sha256_16']}\n")
        for k, v in d.items():
            fh.write(f"{k}: {v}\n")
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
