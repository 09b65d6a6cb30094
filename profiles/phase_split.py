"""Attribute one decode's ncu launch list to phases (trunk / level t) using
the GR4AD_TRACE gemm order of the same command.

    python profiles/phase_split.py launches.csv trace.txt
Prints, for the LAST complete decode in the launch list: per phase and per
kernel name, launches, summed gpu time (us) and DRAM bytes."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ii, ki = h.index("ID"), h.index("Kernel Name")
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    ker = collections.OrderedDict()
    for r in rows[hi + 1:]:
        k = ker.setdefault(int(r[ii]), {"name": r[ki], "t": 0.0, "b": 0.0})
        v = float(r[vi].replace(",", ""))
        u = r[ui].lower()
        if r[mi] == "gpu__time_duration.sum":
            k["t"] += v * {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1e-3)
        elif r[mi].startswith("dram__bytes"):
            k["b"] += v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    return list(ker.values())


def short(n):
    n = n.replace("void ", "")
    base = n.split("(")[0].split("<")[0]
    if "gemm_tc_kernel" in base:
        base += "<" + n.split("<", 1)[1].split(">")[0] + ">"
    return base


def main():
    ks = load(sys.argv[1])
    trace = [l for l in open(sys.argv[2]) if l.startswith("gemm_tc ")]
    # decodes start at the context projection GEMM (EPI_BIAS_DUAL / K = feat_dim)
    starts = [i for i, k in enumerate(ks) if "pad_rows" in k["name"]]
    s0 = starts[-1]
    seg = ks[s0:]
    # phase marks: level_input kernels start levels; everything before the
    # first is encode + trunk
    phase, out = "encode+trunk", collections.OrderedDict()
    lvl = 0
    for k in seg:
        if "level_input" in k["name"]:
            phase = f"level{lvl}"
            lvl += 1
        if "collect_results" in k["name"]:
            phase = "collect"
        d = out.setdefault(phase, collections.OrderedDict())
        e = d.setdefault(short(k["name"]), [0, 0.0, 0.0])
        e[0] += 1
        e[1] += k["t"]
        e[2] += k["b"]
    tot = sum(e[1] for d in out.values() for e in d.values())
    for ph, d in out.items():
        pt = sum(e[1] for e in d.values())
        print(f"== {ph}: {pt/1e3:.2f} ms ({100*pt/tot:.1f} %)")
        for n, (c, t, b) in sorted(d.items(), key=lambda kv: -kv[1][1]):
            print(f"   {n[:90]:90s} x{c:3d} {t/1e3:8.3f} ms {b/1e9:8.3f} GB  "
                  f"{(b/1e9)/(t/1e6) if t else 0:7.0f} GB/s")
    print(f"total {tot/1e3:.2f} ms")


main()
