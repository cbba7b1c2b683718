"""Summarise tools/nvlink_ncu.sh captures into one JSON (profiles/ncu_nvlink_r02.json):
per rank and kernel, the mean NVLink TX / RX bytes per launch (ncu's nvltx / nvlrx
counters, 32 B granularity), the launch duration, and TX GB/s against the
measured 770 GB/s peer-copy and the nominal 900 GB/s per direction
(B200_PROFILING.md).

    python tools/ncu_nvlink_summary.py OUT.json gpurun_out/r2/nvl_*.csv
"""
import csv
import io
import json
import re
import statistics
import sys


def parse(path):
    rows = [l for l in open(path) if l.startswith('"')]
    launches = {}
    for row in csv.DictReader(io.StringIO("".join(rows))):
        key = (int(row["ID"]), row["Kernel Name"])
        launches.setdefault(key, {})[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
    out = {}
    for (_, name), m in sorted(launches.items()):
        kind = "exchange_kernel" if "exchange_kernel" in name else "stream_kernel"
        out.setdefault(kind, []).append(m)
    return out


def main():
    dst, files = sys.argv[1], sys.argv[2:]
    res = {"source": "ncu --metrics nvltx__bytes.sum,gpu__time_duration.sum --clock-control none "
                     "--cache-control none (tools/nvlink_ncu.sh; every rank under its own ncu, "
                     "one counter so a single pass, serialised launches); nvltx counts link "
                     "bytes at 32 B granularity, protocol included",
           "peak_gbs_measured": 770.0, "peak_gbs_nominal": 900.0, "captures": []}
    for f in files:
        m = re.search(r"nvl_n(\d+)_(\d+)_([0-9.]+)_rank(\d+)\.csv", f)
        if not m:
            continue
        n, ng, d, rank = int(m[1]), int(m[2]), float(m[3]), int(m[4])
        for kind, ls in parse(f).items():
            tx = statistics.mean(l.get("nvltx__bytes.sum", 0.0) for l in ls)
            dur = statistics.mean(l.get("gpu__time_duration.sum", 0.0) for l in ls) * 1e-9
            res["captures"].append({
                "n": n, "n_g": ng, "d": d, "rank": rank, "kernel": kind, "launches": len(ls),
                "nvltx_bytes": tx,
                "duration_us": dur * 1e6,
                "tx_gbs": tx / dur / 1e9 if dur else None,
                "tx_frac_of_measured": tx / dur / 770e9 if dur else None})
    json.dump(res, open(dst, "w"), indent=1)
    for c in res["captures"]:
        print(f"n={c['n']} n_g={c['n_g']} d={c['d']} rank {c['rank']} {c['kernel']:16s} "
              f"tx {c['nvltx_bytes'] / 1e6:9.3f} MB "
              f"{c['duration_us']:9.1f} us -> {c['tx_gbs'] or 0:7.1f} GB/s "
              f"({(c['tx_frac_of_measured'] or 0) * 100:.1f}% of 770)")


if __name__ == "__main__":
    main()
