"""Per-region instruction / stall-sample shares of a tile_kernel ncu report
(source view): regions are the kernel's lambdas and phases, found by the
marker lines in csrc/vxb_tile.cuh.
    python tools/ncu_regions.py report.ncu-rep"""
import csv
import subprocess
import sys
from pathlib import Path

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = (Path(__file__).resolve().parents[1] / "paper_2308_01241_b200/csrc/vxb_tile.cuh").read_text().splitlines()
marks = [("noise lambda", "auto noise_chunk = "), ("wait/bucketed", "auto bucketed = "),
         ("consume", "auto consume = "), ("scan_remote", "auto scan_remote = "),
         ("tally", "auto tally = "), ("U (update)", "// ------------------------------------------------ U (update)"),
         ("B (bucketing)", "// ------------------------------------------------ B (bucketing)"),
         ("phase end", "// phase end (CTA-local)"), ("after loop", "// the pending tile P(S(t_last)) back")]
starts = []
for name, m in marks:
    for k, l in enumerate(src, 1):
        if m in l:
            starts.append((k, name))
            break
starts.sort()


def region(f, line):
    if f != "vxb_tile.cuh":
        return "device fns (" + f + ")"
    r = "kernel prologue"
    for k, name in starts:
        if line >= k:
            r = name
    return r


agg = {}
f = None
hdr = None
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] and len(r) > 8 and r[2] == "-":
        try:
            ln, st, ins = int(r[0]), int(r[4]), int(r[7])
        except ValueError:
            continue
        g = region(f, ln)
        a = agg.setdefault(g, [0, 0])
        a[0] += st
        a[1] += ins
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
for g, (st, ins) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{g:28s} stall samples {100 * st / ts:5.1f}%   instructions {100 * ins / ti:5.1f}%")
