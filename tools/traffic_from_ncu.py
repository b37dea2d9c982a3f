"""Per-stage DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
one FastPoint step from an ncu --set full capture of tools/profile_step.py:
kernels in launch order mapped to the bench's stages (the first fps_spec
launch is the prefix, the later FPS launch the early-termination tail)."""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    stages = {}
    seen_fps = False
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if "fps" in name:
            st = "early_term" if seen_fps else "fps_prefix"
            seen_fps = True
        elif "thresholds" in name:
            st = "thresholds"
        elif "grid_" in name or "excl" in name:
            st = "excl_build"
        elif "samp" in name:
            st = "sampler"
        elif "et_" in name:
            st = "early_term"
        elif "bq_rf" in name:
            st = "rf_ball_query"
        else:
            continue
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[k]].replace(",", "") or 0) * scale.get(units[col[k]], 1)
        stages[st] = stages.get(st, 0.0) + b
    stages["source"] = f"ncu --set full of tools/profile_step.py ({rep}), dram__bytes_read.sum + dram__bytes_write.sum per stage"
    json.dump(stages, open(out, "w"), indent=1)
    print(json.dumps(stages, indent=1))


if __name__ == "__main__":
    main()
