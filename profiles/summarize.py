"""Summaries of ncu reports / launch lists for profiles/ (run in the build container)."""
import collections, csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")][:90]
        print(f"## {name}")
        for k in KEYS + [n for n in h if "pipe_tc" in n or "tensor_op" in n][:6]:
            if k in h:
                i = h.index(k)
                print(f"  {k:70s} {v[i]:>16s} {u[i]}")


def _scale(v, unit):
    unit = unit.lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}
    return v * mult.get(unit, 1)


def launch_traffic(path):
    """{kernel: (launches, mean dram bytes per launch)} from a launch list
    captured with dram__bytes_{read,write}.sum (ncu --csv, one row per metric)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ii, ki = h.index("ID"), h.index("Kernel Name")
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.defaultdict(float)
    name_of = {}
    for r in rows[hi + 1:]:
        if r[mi].startswith("dram__bytes"):
            per[r[ii]] += _scale(float(r[vi].replace(",", "")), r[ui])
            name_of[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("<")[0]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, b in per.items():
        agg[name_of[k]][0] += 1
        agg[name_of[k]][1] += b
    return {k: (n, b / n) for k, (n, b) in agg.items()}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        name = name.split("<")[0]
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("ns", "nsecond") else (v * 1e3 if r[ui] in ("ms", "msecond") else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(x[1] for x in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'us':>12s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} {n:8d} {t:12.1f} {100 * t / tot:6.1f}%")
    print(f"total {sum(x[0] for x in agg.values())} launches, {tot:.1f} us (cold, serialised)")


def write_traffic(out, **lists):
    """profiles/traffic.json: per config, the mean DRAM bytes per launch of
    each kernel (bench.py reports it as roofline.traffic)."""
    import json
    data = {}
    for cfg, path in lists.items():
        data[cfg] = {k: {"launches": n, "dram_bytes_per_launch": b, "source": path}
                     for k, (n, b) in launch_traffic(path).items()}
    with open(out, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    if sys.argv[1] == "--traffic":
        write_traffic(sys.argv[2], **dict(a.split("=", 1) for a in sys.argv[3:]))
        sys.exit(0)
    for p in sys.argv[1:]:
        print(f"# {p}")
        (report if p.endswith(".ncu-rep") else launches)(p)
        print()
