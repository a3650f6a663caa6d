"""Summarise an ncu report (read here, no GPU): key raw metrics per kernel and the
per-function split of warp-stall samples / executed instructions from the SASS page.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"== kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
        stalls = sorted(((float(d[k] or 0), k) for k in hdr
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")),
                        reverse=True)[:8]
        print("  top stall reasons (warps per issue-active cycle):")
        for v, k in stalls:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")
    agg, fn, h = {}, None, None
    for row in csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))):
        if not row:
            continue
        if row[0] == "Kernel Name":
            fn = row[1]
            continue
        if row[0] == "Address":
            h = row
            continue
        d = dict(zip(h, row))
        a = agg.setdefault(fn, [0, 0])
        try:
            a[0] += int(d["Warp Stall Sampling (All Samples)"])
            a[1] += int(d["Instructions Executed"])
        except (KeyError, ValueError):
            pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print("== per-function split (SASS source page): % of stall samples, % of warp instructions")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"  {100 * v[0] / ts:5.1f}%  {100 * v[1] / ti:5.1f}%  {k[:140]}")


if __name__ == "__main__":
    main(sys.argv[1])
