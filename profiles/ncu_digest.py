"""One line per ncu --set full capture (raw page CSV): kernel, duration, SM
clock, DRAM bytes and throughput, tensor pipe activity, issue slots,
occupancy, top stall reasons.

    python profiles/ncu_digest.py gpurun_out/ev/prof_*.raw.csv > profiles/r2/ncu_summary.txt"""
import csv
import sys

KEYS = [("us", "gpu__time_duration.sum"),
        ("sm_ghz", "smsp__cycles_elapsed.avg.per_second"),
        ("dram_rd", "dram__bytes_read.sum"), ("dram_wr", "dram__bytes_write.sum"),
        ("dram_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("utchmma_ops_pct", "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
        ("hmma_inst_pct", "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"),
        ("l2_pct", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
        ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("warps_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
        ("block", "launch__block_size")]


def main(paths):
    for p in paths:
        rows = list(csv.reader(open(p)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        print(f"## {p.split('/')[-1].replace('.raw.csv', '')}: {name[:110]}")
        parts = []
        for label, k in KEYS:
            if k in d and d[k] != "":
                parts.append(f"{label}={d[k]}{(' ' + u[k]) if u.get(k) and u[k] not in ('', '%') else ''}")
        print("   " + "  ".join(parts))
        st = {k: v for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled")
              and not k.endswith("not_issued") and v}
        tot = sum(float(v.replace(",", "")) for v in st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -float(kv[1].replace(",", "")))[:6]
        print("   stalls: " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v.replace(',', '')) / tot:.0f}%"
            for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1:])
