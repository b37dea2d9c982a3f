"""Aggregate ncu warp-stall samples per CUDA source line.

  python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, path = [], ""
    H = None
    for r in rows:
        if r and r[0] == "File Path":
            path = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            H = r
            continue
        if H and r and r[0] not in ("-", "File Path", "Function Name") and len(r) > 4:
            try:
                res.append((float(r[4]), f"{path}:{r[0]}", r[1][:100]))
            except ValueError:
                pass
    tot = sum(x[0] for x in res) or 1
    for v, loc, src in sorted(res, reverse=True)[:top]:
        print(f"{100 * v / tot:5.1f}%  {loc:18s} {src}")


if __name__ == "__main__":
    main()
