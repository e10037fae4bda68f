"""Summarise an ncu --set full report (.ncu-rep) per kernel launch into JSON:
duration, DRAM bytes read / written, achieved DRAM GB/s and its fraction of
the measured HBM peak (MEASURED_PEAKS.json hbm_gbs), L2 hit rate, FP64 pipe
activity, registers, occupancy and the top warp-stall reasons (PC sampling).
Usage: python scripts/ncu_summary.py report.ncu-rep [--algorithmic-bytes B]
       [--label text] > profiles/<name>.json"""
import argparse
import csv
import io
import json
import os
import subprocess

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
         "nsecond": 1e-9}


def hbm_peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))["hbm_gbs"]
    except Exception:  # noqa: BLE001
        return 6545.6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--algorithmic-bytes", type=float, default=None, help="algorithmic bytes per launch")
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    peak = hbm_peak()
    res = {"report": os.path.basename(a.report), "label": a.label, "hbm_peak_gbs_measured": peak, "launches": []}
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))

        def val(k):
            try:
                return float(d[k].replace(",", "")) * SCALE.get(u.get(k, ""), 1.0)
            except (KeyError, ValueError):
                return None
        t = val("gpu__time_duration.sum")
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        stalls = {}
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(d[k]))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda x: -x[1])[:6]
        L = {"kernel": d.get("Kernel Name", "")[:120], "duration_s": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
             "dram_gbs": (rd + wr) / t / 1e9 if t and rd is not None else None,
             "l2_hit_pct": val("lts__t_sector_hit_rate.pct"),
             "fp64_pipe_active_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
             "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
             "registers": val("launch__registers_per_thread"), "grid": val("launch__grid_size"),
             "block": val("launch__block_size"),
             "top_stalls_pct": {k: round(100.0 * v / tot, 1) for k, v in top}}
        if L["dram_gbs"]:
            L["dram_frac_of_measured_hbm"] = L["dram_gbs"] / peak
        if a.algorithmic_bytes and t:
            L["algorithmic_bytes"] = a.algorithmic_bytes
            L["algorithmic_gbs"] = a.algorithmic_bytes / t / 1e9
            L["algorithmic_frac_of_measured_hbm"] = L["algorithmic_gbs"] / peak
        res["launches"].append(L)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
