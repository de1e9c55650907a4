"""Summarise an ncu report: per kernel key metrics (+ top stall reasons)."""
import csv
import io
import re
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_rd_MB",
    "dram__bytes_write.sum": "dram_wr_MB",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "inst",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64pipe%",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64inst%",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conf",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "st_longsb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "st_barrier",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "st_shortsb",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "st_wait",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "st_mathpipe",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio": "st_noinst",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "st_mio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "st_lg",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio": "st_dispatch",
    "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio": "st_tex",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio": "st_drain",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio": "st_membar",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio": "st_branch",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio": "st_selected",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio": "st_notsel",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = re.sub(r"\(.*", "", d.get("Kernel Name", ""))[:70]
        vals = {}
        unit_of = dict(zip(hdr, units))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,  # -> us
                 "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}          # -> MB
        for k, short in WANT.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    vals[short] = float(d[k].replace(",", "")) * scale.get(unit_of.get(k, ""), 1.0)
                except ValueError:
                    pass
        stalls = sorted(((v, k) for k, v in vals.items() if k.startswith("st_")), reverse=True)[:5]
        base = {k: v for k, v in vals.items() if not k.startswith("st_")}
        print(name)
        print("   ", {k: round(v, 2) for k, v in base.items()})
        print("    stalls:", ", ".join(f"{k}={v:.2f}" for v, k in stalls))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
