#!/usr/bin/env python
"""Summarise an .ncu-rep: key throughput metrics, stall reasons, top stalled SASS lines."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def main(rep, top=25):
    h, data = raw(rep)
    for d in data:
        v = dict(zip(h, d))
        print("kernel:", v.get("Kernel Name", "")[:100])
        for k in KEYS:
            if k in v:
                print(f"  {k:70s} {v[k]}")
        st = [(k, float(x)) for k, x in v.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and x not in ("", "n/a")]
        st.sort(key=lambda t: -t[1])
        print("  stalls (warps per issue):", ", ".join(f"{k[34:-23]}={x:.2f}" for k, x in st[:8]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2:
        hh = rows[1]
        iS, iSrc, iE = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source"), hh.index("Instructions Executed")
        dd = [r for r in rows[2:] if len(r) > iS and r[iS].replace('.', '', 1).isdigit()]
        tot = sum(float(r[iS] or 0) for r in dd) or 1
        print(f"  top stalled SASS ({tot:.0f} samples):")
        for r in sorted(dd, key=lambda r: -float(r[iS] or 0))[:top]:
            print(f"   {100*float(r[iS] or 0)/tot:5.1f}%  exec={r[iE]:>8}  {r[iSrc][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
