"""Summarise an ncu report: headline metrics + top stall sites (SASS) with
their source lines.  python tools/ncu_summary.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
        "lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum",
        "lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum",
        "lts__d_atomic_input_cycles_active.sum.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    h, u, v = rows[0], rows[1], rows[2]
    for name in WANT:
        if name in h:
            i = h.index(name)
            print(f"{name:70s} {v[i]:>18s} {u[i]}")
    sass = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv",
                                             "--print-source", "sass"]))))
    hh = sass[1]
    data = sass[2:]
    si = hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in data if r[si].isdigit())
    print(f"\nstall samples: {tot}")
    order = sorted(range(len(data)), key=lambda k: -int(data[k][si]) if data[k][si].isdigit() else 0)
    for k in order[:top]:
        r = data[k]
        print(f"{k:5d} {int(r[si]) / tot * 100:6.2f}%  {r[1][:90]}")


if __name__ == "__main__":
    main()
