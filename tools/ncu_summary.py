"""Text summary of one kernel in an `ncu --set full` report (the format of profiles/r*_gather_ncu.txt,
which bench.py's gather_capture() parses): key raw metrics, warp-stall sampling, instruction mix.

    python tools/ncu_summary.py REPORT.ncu-rep "header line" > profiles/rNN_gather_ncu.txt
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def ncu_csv(rep, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", *extra], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main():
    rep, header = sys.argv[1], sys.argv[2]
    extra = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    h, units, vals = ncu_csv(rep, *extra)
    d, u = dict(zip(h, vals)), dict(zip(h, units))
    print(f"# {header}")
    print(f"Kernel Name{' ' * 66}{d['Kernel Name']} ")
    for m in METRICS:
        if m in d:
            print(f"{m:<76}{d[m]} {u.get(m, '')}".rstrip())
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1.0
    print("\n# warp stall sampling (all samples)")
    for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
        print(f"  {100 * v / tot:5.1f}%  {k}")
    h2, _, v2 = ncu_csv(rep, *extra, "--print-metric-instances", "details", "--metrics",
                        "sass__inst_executed_per_opcode")
    txt = dict(zip(h2, v2)).get("sass__inst_executed_per_opcode", "")
    m = re.match(r"\s*(\d+)\s*\((.*)\)", txt)
    if m:
        total = int(m.group(1))
        print("\n# executed instruction mix (warp-level)")
        for part in m.group(2).split(";")[:10]:
            op, cnt = part.split(":")
            print(f"  {op.strip():<16}{int(cnt):>10}  {100 * int(cnt) / total:4.1f}%")


if __name__ == "__main__":
    main()
