"""Key per-kernel metrics from an `ncu --page raw --csv` export (one line per launch)."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "blk"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dsmem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("lts__t_sector_hit_rate.pct", "L2hit%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("smsp__inst_executed.sum", "winst"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall_lsb"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb/iss"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "bar/iss"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "ssb/iss"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "wait/iss"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "math/iss"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "lgthr/iss"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "mio/iss"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "noinst/iss"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "membar/iss"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "br/iss"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "disp/iss"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "lg/iss"),
    ("smsp__average_warps_issue_stalled_selected_per_issue_active.ratio", "sel/iss"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "nsel/iss"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "drain/iss"),
    ("smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio", "imc/iss"),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "sleep/iss"),
    ("dram__bytes_read.sum", "dramR"),
    ("dram__bytes_write.sum", "dramW"),
]


def main(path, pattern=""):
    rows = list(csv.reader(open(path)))
    # ncu's own ==PROF== / ==WARNING== lines (and anything the profiled program
    # printed) come before the CSV header when stdout was captured whole
    while rows and "Kernel Name" not in rows[0]:
        rows.pop(0)
    if len(rows) < 2:
        sys.exit(f"{path}: no ncu raw-page CSV header found")
    hdr = rows[0]
    units = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    kcol = col.get("Kernel Name")
    for r in rows[2:]:
        name = r[kcol] if kcol is not None else "?"
        if pattern and pattern not in name:
            continue
        out = [name[:60]]
        for k, short in KEYS:
            if k in col and r[col[k]] not in ("", "n/a"):
                v = r[col[k]].replace(",", "")
                u = units[col[k]]
                try:
                    x = float(v)
                    if k == "gpu__time_duration.sum":
                        x = x / 1000.0 if u == "ns" else (x * 1000.0 if u == "ms" else x)
                    out.append(f"{short}={x:.4g}")
                except ValueError:
                    out.append(f"{short}={v}")
        print(" ".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
