"""Key metrics per launch from `ncu -i REP --page raw --csv` output.

    python profiles/ncu_raw.py gpurun_out/x_raw.csv"""
import csv
import sys

WANT = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:70])
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"    {w:70s} {r[i]:>14s} {units[i]}")
