"""Top source lines by warp-stall samples from an ncu report (cuda+sass view).
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, lines, hdr = None, [], None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0] not in ("", "Function Name") and r[0].isdigit():
            si = hdr.index("Warp Stall Sampling (All Samples)")
            try:
                lines.append((int(r[si]), fname, int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    for n, f, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * n / tot:6.2f}%  {f}:{ln:<5d} {src[:100]}")


if __name__ == "__main__":
    main()
