"""Summarise one kernel of an ncu --set full report into a small text file for profiles/.
Usage: python tools/ncu_summary.py report.ncu-rep out.txt [title]"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg", "sm__cycles_active.max",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, vals = rows[0], rows[1], rows[2]
    name = vals[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    lines = [f"# {title}", f"kernel: {name}"]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"{k:70s} {vals[i]:>16s} {units[i]}")
    stalls = [(h[i], vals[i]) for i in range(len(h))
              if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
    stalls = sorted(stalls, key=lambda x: -float(x[1].replace(",", "") or 0))[:8]
    lines.append("top warp-stall samples:")
    lines += [f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {v}" for k, v in stalls]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
