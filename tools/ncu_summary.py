"""Summarise ncu --set full reports (read here, no GPU): per kernel launch the
duration, DRAM bytes, L2 hit rate, issue activity and the top warp-stall
reasons per issued instruction.  Usage: python tools/ncu_summary.py rep.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "long_scoreboard_per_issue",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "barrier_per_issue",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "short_scoreboard_per_issue",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "wait_per_issue",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio": "membar_per_issue",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio": "branch_resolving_per_issue",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "math_throttle_per_issue",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "mio_throttle_per_issue",
}


def _num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return x


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for k, name in WANT.items():
            if k in hdr:
                v = _num(r[hdr.index(k)])
                u = units[hdr.index(k)]
                if u == "Kbyte":
                    v *= 1e3
                elif u == "Mbyte":
                    v *= 1e6
                elif u == "Gbyte":
                    v *= 1e9
                elif u in ("us", "usecond"):
                    v *= 1e3
                elif u in ("ms", "msecond"):
                    v *= 1e6
                d[name] = v
        if "dram_read" in d:
            d["dram_bytes"] = d["dram_read"] + d.get("dram_write", 0.0)
        res.append(d)
    return res


if __name__ == "__main__":
    print(json.dumps({p: summarise(p) for p in sys.argv[1:]}, indent=1))
