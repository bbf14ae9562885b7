"""Key counters of an `ncu --set full` report (one or more kernels):
time, DRAM bytes and throughput, occupancy, L1/smem pressure and the
sampled stall reasons.  usage: python scripts/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        print(f"== {d.get('Kernel Name')} grid {d.get('launch__grid_size')}")
        for k in KEYS:
            print(f"   {k:60s} {d.get(k)}")
        st = sorted(((int(float(v)), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k, v in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v),
                    reverse=True)
        print("   stalls:", ", ".join(f"{n} {c}" for c, n in st[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
