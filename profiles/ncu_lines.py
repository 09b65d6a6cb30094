"""Per-source-line stall summary from `ncu -i REP --page source --csv
--print-source cuda,sass` output (kernels built with -lineinfo).

    python profiles/ncu_lines.py gpurun_out/srcsass.csv [top_n]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, cur_file, hdr = [], None, None
with open(path, newline="") as fh:
    for r in csv.reader(fh):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        rec = dict(zip(hdr[2:], r[2:]))
        try:
            samp = int(rec["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        stalls = {k[6:]: int(v) for k, v in rec.items()
                  if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
        inst = int(rec.get("Instructions Executed", "0") or 0)
        rows.append((samp, cur_file, r[0], r[1].strip()[:70], inst, stalls))
total = sum(x[0] for x in rows)
tinst = sum(x[4] for x in rows)
print(f"total samples {total}, warp-instructions {tinst}")
for samp, f, ln, src, inst, st in sorted(rows, key=lambda x: -x[0])[:top]:
    s3 = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{100 * samp / total:5.1f}% {f}:{ln:5s} inst {inst:9d}  [{s3}]  {src}")
