"""One line per kernel launch of an ncu report: duration, DRAM GB/s and % of peak, tensor / FP64 /
FMA pipe activity, L1 data-pipe load, achieved occupancy.

    python tools/ncu_table.py REPORT.ncu-rep "header" > profiles/rNN_xxx_ncu.txt
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("us", "gpu__time_duration.sum", 1e-3),
    ("dram_MB", None, None),
    ("dram_TB/s", None, None),
    ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("tensor%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("fma%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    ("l1pipe%", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("occ%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    ("smem_confl", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
]


def main():
    rep, header = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    u = dict(zip(h, units))
    print(f"# {header}")
    print(f"# {'kernel':<44}" + "".join(f"{c[0]:>11}" for c in COLS) + "  grid x block")
    for r in rows[2:]:
        d = dict(zip(h, r))

        def num(k):
            try:
                return float(d.get(k, "") or "nan")
            except ValueError:
                return float("nan")
        us = num("gpu__time_duration.sum") * (1e-3 if u.get("gpu__time_duration.sum") == "ns" else 1.0)
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        mb = (num("dram__bytes_read.sum") * scale.get(u.get("dram__bytes_read.sum"), 1.0)
              + num("dram__bytes_write.sum") * scale.get(u.get("dram__bytes_write.sum"), 1.0))
        vals = [us, mb, mb / us if us > 0 else float("nan")]  # MB / us = TB/s
        for _, key, _s in COLS[3:]:
            vals.append(num(key))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:44]
        print(f"  {name:<44}" + "".join(f"{v:>11.1f}" for v in vals)
              + f"  {d.get('launch__grid_size', '?')} x {d.get('launch__block_size', '?')}")


if __name__ == "__main__":
    main()
