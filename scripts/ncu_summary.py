"""Summarise an ncu --set full report (read here, no GPU) into profiles/.

usage: python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<name>.md [dtype-key]
Writes the markdown summary and, with a dtype key, updates
profiles/traffic.json (DRAM bytes per launch, read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__inst_executed.sum", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_membar",
    "smsp__pcsamp_warps_issue_stalled_sleeping", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_drain",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu summary: {os.path.basename(rep)}", "",
             "| launch | kernel | metric | value | unit |", "|---|---|---|---|---|"]
    traffic = None
    ki = hdr.index("Kernel Name")
    for li, v in enumerate(rows[2:]):
        d = {n: (v[i], units[i]) for i, n in enumerate(hdr)}
        for w in WANT:
            if w in d:
                lines.append(f"| {li} | {v[ki][:40]} | {w} | {d[w][0]} | {d[w][1]} |")
        rb = float(d["dram__bytes_read.sum"][0].replace(",", ""))
        wb = float(d["dram__bytes_write.sum"][0].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = rb * scale[d["dram__bytes_read.sum"][1]] + wb * scale[d["dram__bytes_write.sum"][1]]
        lines.append(f"| {li} | | dram read+write (bytes) | {traffic:.0f} | byte |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if key and traffic is not None:
        p = os.path.join(os.path.dirname(out), "traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[key] = traffic
        d[f"{key}_source"] = os.path.basename(rep)
        json.dump(d, open(p, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
