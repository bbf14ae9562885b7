"""Per-kernel table of one cfg-2 program step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file ... python bench.py --steps 1 --warmup 1`): the first
complex64 program launch (K2 small_kernel stages, K1 large_kernel items, K4
k4_kernel expansion items),
durations and DRAM bytes per kernel, cold-cache and serialised by ncu.

usage: python scripts/launch_summary.py nodes.csv [graph.csv] > profiles/<name>.md"""
import csv
import re
import sys


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = list(csv.reader(lines))
    h = r[0]
    out = {}
    order = []
    for row in r[1:]:
        d = dict(zip(h, row))
        key = d["ID"]
        if key not in out:
            out[key] = {"name": d["Kernel Name"], "grid": d["Grid Size"]}
            order.append(key)
        v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
        out[key][d["Metric Name"]] = v * scale
    return [out[k] for k in order]


def short(name):
    m = re.search(r"(large_kernel_c64|large_kernel_c128|large_kernel|small_kernel|k4_kernel|k3v2_kernel)<([^>]*)>", name)
    return f"{m.group(1)}<{m.group(2).replace('(int)', '')}>" if m else name[:60]


def main():
    ks = rows(sys.argv[1])
    fam = ("large_kernel_c64<", "large_kernel<float", "small_kernel<float", "k4_kernel<float", "k3v2_kernel<float")
    ours = [k for k in ks if any(f in k["name"] for f in fam)]
    # the first program launch: its node count (bench.py config.program.nodes)
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 21
    step = ours[:n]
    tot_t = sum(k["gpu__time_duration.sum"] for k in step)
    tot_b = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in step)
    print("# cfg-2 lightcone, one complex64 program step: per-kernel ncu launch list\n")
    print("Source: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none` of `bench.py --steps 1 --warmup 1` (graph nodes profiled one by one: "
          "cold L2, serialised; shares, not absolute times, compare with the live bench).\n")
    print("| # | kernel | grid | us | DRAM read MB | DRAM write MB | GB/s | share of step |")
    print("|---|---|---|---|---|---|---|---|")
    for i, k in enumerate(step):
        t = k["gpu__time_duration.sum"]
        b = k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        print(f"| {i} | {short(k['name'])} | {k['grid']} | {t * 1e6:.1f} | {k['dram__bytes_read.sum'] / 1e6:.1f} | "
              f"{k['dram__bytes_write.sum'] / 1e6:.1f} | {b / t / 1e9:.0f} | {100 * t / tot_t:.1f}% |")
    print(f"\nSum: {tot_t * 1e6:.1f} us serialised, {tot_b / 1e9:.3f} GB DRAM.")
    dom = max(step, key=lambda k: k["gpu__time_duration.sum"])
    print(f"Dominant kernel: {short(dom['name'])}, {100 * dom['gpu__time_duration.sum'] / tot_t:.1f}% of the "
          f"serialised step.")
    if len(sys.argv) > 2 and sys.argv[2] != "-":
        g = rows(sys.argv[2])
        g = [k for k in g if k["name"] == "graph" and "dram__bytes_read.sum" in k]
        if g:
            # graph-level profiling: one row per graph launch; the first is the first c64 step
            k = g[0]
            b = k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
            print(f"\nWhole graph (ncu --graph-profiling graph, first launch): {k['gpu__time_duration.sum'] * 1e6:.1f} us, "
                  f"DRAM {b / 1e9:.3f} GB (read {k['dram__bytes_read.sum'] / 1e9:.3f}, write "
                  f"{k['dram__bytes_write.sum'] / 1e9:.3f}).")


if __name__ == "__main__":
    main()
