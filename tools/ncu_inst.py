"""Executed warp instructions per source line from an ncu report (cuda,sass
view): where the instruction budget of a kernel goes.
python tools/ncu_inst.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    fname, ie, lines, perfile = None, None, [], collections.Counter()
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            ie = r.index("Instructions Executed")
        elif ie is not None and len(r) > ie and r[0].isdigit():
            try:
                v = int(float(r[ie]))
            except ValueError:
                continue
            if v:
                lines.append((v, fname, r[0], r[1][:90]))
                perfile[fname] += v
    tot = sum(v for v, *_ in lines)
    print(f"total warp instructions {tot:.4g}:",
          ", ".join(f"{k} {v / tot:.1%}" for k, v in perfile.most_common()))
    for v, f, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{v / tot:6.2%}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
