"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) per (kernel, grid):
total ms, launches, mean us, DRAM MB read / written per launch.

    python profiles/launch_list.py gpurun_out/x/launches_c3.csv > profiles/r2/launches_c3.txt"""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}

acc = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = (d["Kernel Name"][:72], d["Grid Size"])
    v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    m = d["Metric Name"]
    if m == "gpu__time_duration.sum":
        acc[k][0] += 1
        acc[k][1] += v  # us
    elif m == "dram__bytes_read.sum":
        acc[k][2] += v
    elif m == "dram__bytes_write.sum":
        acc[k][3] += v
tot = sum(a[1] for a in acc.values())
print("# total_ms  share  launches  mean_us  dram_read_MB/launch  dram_write_MB/launch  kernel  grid")
for (name, grid), (n, t, rd, wr) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    n = max(n, 1)
    print(f"{t / 1e3:9.3f} {100 * t / tot:5.1f}% {n:5d} {t / n:9.1f} {rd / n / 1e6:9.1f} "
          f"{wr / n / 1e6:9.1f}  {name}  {grid}")
