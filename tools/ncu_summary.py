"""Summarise an ncu --set full report (key roofline metrics + top stall sites).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [n_top]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"== {name[:120]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:70s} {r[i]:>14s} {u[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        hh = src[1]
        si = hh.index("Warp Stall Sampling (All Samples)")
        data = [r for r in src[2:] if len(r) > si and r[si].isdigit()]
        tot = sum(int(r[si]) for r in data) or 1
        print(f"  top stall sites ({tot} samples):")
        for r in sorted(data, key=lambda r: -int(r[si]))[:ntop]:
            print(f"    {int(r[si]) / tot * 100:5.1f}%  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
