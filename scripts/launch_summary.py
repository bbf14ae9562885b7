"""Per-kernel table of ONE cfg-2 program step from an ncu launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file nodes.csv \
        python scripts/one_step.py c128          # exactly one program launch
    python scripts/launch_summary.py nodes.csv <n_nodes> [c128|c64] > profiles/<name>.md

Every kernel of this library is matched (K2 small_kernel, K1
large_kernel_c64/_c128, K3 k3_kernel/k3v2_kernel, K4 k4_kernel_c64/_c128, K5
k5_kernel_c64/_c128, K6 k6_kernel_c64/_c128);
the first <n_nodes> of them are the step (scripts/one_step.py prints the
program's node count).  Times are ncu's: cold L2, serialised node by node —
the SHARE of each kernel is what compares with the live bench."""
import csv
import re
import sys

FAMILIES = r"(small_kernel|large_kernel_c64|large_kernel_c128|k3v2_kernel|k3_kernel|k4_kernel_c64|k4_kernel_c128|k5_kernel_c64|k5_kernel_c128|k6_kernel_c64|k6_kernel_c128)"
FAMILY_OF = {"small_kernel": "K2", "large_kernel_c64": "K1", "large_kernel_c128": "K1", "k3v2_kernel": "K3",
             "k3_kernel": "K3", "k4_kernel_c64": "K4", "k4_kernel_c128": "K4", "k5_kernel_c64": "K5",
             "k5_kernel_c128": "K5", "k6_kernel_c64": "K6", "k6_kernel_c128": "K6"}


def rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    r = list(csv.reader(lines))
    h = r[0]
    out, order = {}, []
    for row in r[1:]:
        d = dict(zip(h, row))
        key = d["ID"]
        if key not in out:
            out[key] = {"name": d["Kernel Name"], "grid": d["Grid Size"]}
            order.append(key)
        v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(d["Metric Unit"], 1.0)
        out[key][d["Metric Name"]] = v * scale
    return [out[k] for k in order]


def family(name):
    m = re.search(FAMILIES + r"\b", name)
    return m.group(1) if m else None


def short(name):
    m = re.search(FAMILIES + r"(<[^()]*>)?", name)
    return (m.group(1) + (m.group(2) or "")).replace("(int)", "") if m else name[:60]


def main():
    ks = rows(sys.argv[1])
    n = int(sys.argv[2])
    dt = sys.argv[3] if len(sys.argv) > 3 else "c128"
    ours = [k for k in ks if family(k["name"])]
    step = ours[:n]
    assert len(step) == n, f"launch list holds {len(step)} of our kernels, expected {n}"
    tot_t = sum(k["gpu__time_duration.sum"] for k in step)
    tot_b = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in step)
    print(f"# cfg-2 lightcone, one {dt} program step: per-kernel ncu launch list\n")
    print("Source: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none` of `scripts/one_step.py` (exactly one program launch; graph nodes profiled one by "
          "one: cold L2, serialised — shares, not absolute times, compare with the live bench).\n")
    print("| # | family | kernel | grid | us | DRAM read MB | DRAM write MB | GB/s | share of step |")
    print("|---|---|---|---|---|---|---|---|---|")
    for i, k in enumerate(step):
        t = k["gpu__time_duration.sum"]
        rd, wr = k.get("dram__bytes_read.sum", 0), k.get("dram__bytes_write.sum", 0)
        print(f"| {i} | {FAMILY_OF[family(k['name'])]} | {short(k['name'])} | {k['grid']} | {t * 1e6:.1f} | "
              f"{rd / 1e6:.1f} | {wr / 1e6:.1f} | {(rd + wr) / t / 1e9:.0f} | {100 * t / tot_t:.1f}% |")
    print(f"\nSum: {tot_t * 1e6:.1f} us serialised, {tot_b / 1e9:.3f} GB DRAM.")
    dom = max(step, key=lambda k: k["gpu__time_duration.sum"])
    print(f"Dominant kernel: {FAMILY_OF[family(dom['name'])]} {short(dom['name'])}, "
          f"{100 * dom['gpu__time_duration.sum'] / tot_t:.1f}% of the serialised step.")


if __name__ == "__main__":
    main()
