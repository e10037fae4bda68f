"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, summed durations and shares of the library's
kernel time.  Usage: launch_shares.py launches.csv source-description > out.json"""
import csv
import json
import re
import sys
from collections import OrderedDict


def base_name(full):
    s = re.sub(r"^void\s+", "", full)
    s = s.split("(")[0] if not s.startswith("<") else s
    # drop template arguments (nested), keep the qualified identifier
    out, depth = [], 0
    for ch in s:
        if ch == "<":
            depth += 1
            continue
        if ch == ">":
            depth -= 1
            continue
        if depth == 0:
            out.append(ch)
    name = "".join(out).replace("unnamed::", "").strip(":")
    return name.split("::")[-1] or full[:60]


def main():
    path, src = sys.argv[1], sys.argv[2]
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    ours, other = OrderedDict(), {"launches": 0, "ms": 0.0}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            ns *= 1e3
        elif r["Metric Unit"] == "ms":
            ns *= 1e6
        full = r["Kernel Name"]
        if "at::" in full or "at_cuda" in full or full.startswith("void at") or "cub::" in full:
            other["launches"] += 1
            other["ms"] += ns / 1e6
            continue
        b = base_name(full)
        e = ours.setdefault(b, {"launches": 0, "ms": 0.0, "example": full[:160]})
        e["launches"] += 1
        e["ms"] += ns / 1e6
    tot = sum(v["ms"] for v in ours.values())
    for v in ours.values():
        v["share"] = v["ms"] / tot if tot else 0.0
    ours = OrderedDict(sorted(ours.items(), key=lambda kv: -kv[1]["ms"]))
    print(json.dumps({"source": src, "total_ms_ebv_kernels": tot,
                      "ebv_launches": sum(v["launches"] for v in ours.values()),
                      "kernels": ours, "torch_kernels": other}, indent=1))


if __name__ == "__main__":
    main()
