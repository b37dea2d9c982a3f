"""Summarise an ncu --set full report: per kernel launch duration, DRAM
traffic, throughput, occupancy and the top warp-stall reasons."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    col = {k: i for i, k in enumerate(h)}

    def g(r, k):
        return r[col[k]] if k in col else ""

    for r in rows[2:]:
        name = g(r, "Kernel Name").split("(")[0].replace("void ", "").replace("ps::<unnamed>::", "")
        dur_u = rows[1][col["gpu__time_duration.sum"]]
        dur_ns = float(g(r, "gpu__time_duration.sum").replace(",", "") or 0) * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(dur_u, 1)
        rd = float(g(r, "dram__bytes_read.sum").replace(",", "") or 0)
        wr = float(g(r, "dram__bytes_write.sum").replace(",", "") or 0)
        ur = rows[1][col["dram__bytes_read.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
        uw = rows[1][col["dram__bytes_write.sum"]]
        scalew = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uw, 1)
        stalls = [(float(g(r, k).replace(",", "") or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                  for k in col if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(x for x, _ in stalls) or 1
        top = ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(stalls, reverse=True)[:4])
        # achieved DRAM bandwidth against the measured peak, and the units' throughput shares
        dur_s = dur_ns * 1e-9 if dur_ns else 0.0
        gbs = (rd * scale + wr * scalew) / dur_s / 1e9 if dur_s else 0.0
        pk = 6536.0
        try:
            import json
            import os
            pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:  # noqa: BLE001 - fallback peak of the profiling recipe
            pass
        def pct(k):
            v = g(r, k).replace(",", "")
            return f"{float(v):.1f}%" if v else "n/a"
        print(f"{name}: duration {g(r, 'gpu__time_duration.sum')} {rows[1][col['gpu__time_duration.sum']]}; "
              f"DRAM read {rd * scale / 1e6:.2f} MB write {wr * scalew / 1e6:.2f} MB; "
              f"grid {g(r, 'launch__grid_size')} x {g(r, 'launch__block_size')} cluster {g(r, 'launch__cluster_dim_x')}; "
              f"regs {g(r, 'launch__registers_per_thread')}; warps active {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')}%; "
              f"issue active {g(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active')}%; "
              f"inst {g(r, 'smsp__inst_executed.sum')}; "
              f"DRAM {gbs:.0f} GB/s = {100 * gbs / pk:.1f}% of the measured {pk:.0f}; L1/shared "
              f"{pct('l1tex__throughput.avg.pct_of_peak_sustained_elapsed')}, L2 "
              f"{pct('lts__throughput.avg.pct_of_peak_sustained_elapsed')} of peak; stalls: {top}")


if __name__ == "__main__":
    main()
