"""Aggregate ncu source-page metrics per CUDA source line.

  python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [--inst]

Default ranks lines by warp-stall samples; --inst ranks by instructions
executed and also prints the dominant stall reasons of each line.
"""
import csv
import io
import subprocess
import sys


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    rep, kern = args[0], args[1]
    top = int(args[2]) if len(args) > 2 else 25
    by_inst = "--inst" in sys.argv
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, path = [], ""
    H = None
    for r in rows:
        if r and r[0] in ("File Path", "File Name"):
            path = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            H = r
            continue
        if H and r and r[0] not in ("-", "File Path", "File Name", "Function Name") and len(r) > 7:
            try:
                samp = float(r[4] or 0)
                inst = float(r[7] or 0)
            except ValueError:
                continue
            stalls = []
            for k, name in enumerate(H):
                if name.startswith("stall_") and "Not Issued" not in name:
                    try:
                        stalls.append((float(r[k] or 0), name[6:]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            res.append((inst if by_inst else samp, samp, inst, f"{path}:{r[0]}", r[1][:80],
                        ",".join(f"{n}={int(v)}" for v, n in stalls[:3] if v > 0)))
    tot = sum(x[0] for x in res) or 1
    for key, samp, inst, loc, src, st in sorted(res, reverse=True)[:top]:
        print(f"{100 * key / tot:5.1f}%  inst={inst:10.0f} samp={samp:7.0f} {loc:20s} {src}  [{st}]")


if __name__ == "__main__":
    main()
