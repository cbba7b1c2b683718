"""Markdown table of configs[4] sweep lines (tools/sweep.py output).

    python tools/sweep_table.py profiles/sweep_r02_n1.jsonl [more.jsonl ...]
"""
import json
import sys

PEAK = 6551.4


def main():
    rows = []
    for f in sys.argv[1:]:
        for line in open(f):
            d = json.loads(line)
            if "value" not in d:
                continue
            r = d["roofline"]
            ncu = (r.get("ncu") or {}).get("k1") or {}
            cpu = (d.get("cpu_baseline") or {}).get("value")
            nv = d.get("nvlink") or {}
            n_g, dd, n = d["config"]["n_g"], d["config"]["d"], d["n_gpus"]
            es = 8 if d["dtype"] == "f64" else 4
            kp = d["records"]["k_prime_mean"]
            # the step's algorithmic bytes: select/compact 3*T*n_g + (4+T)*k_i,
            # gather/clear + scatter 8*k' (n = 1: the scatter only)
            step_bytes = 3 * es * n_g + (4 + es) * kp / n + (8 if n > 1 else 4 + es) * kp
            rows.append((n, n_g, dd, d["value"] * 1e3, r["kernel_ms"] * 1e3, r["finish_kernel_ms"] * 1e3,
                         r["frac"], ncu.get("dram_frac"), step_bytes / (d["value"] * 1e-3) / 1e9 / PEAK,
                         d["records"]["density_over_d"], nv.get("achieved_gbs"), cpu))
    rows.sort()
    print("| N | n_g | d | step µs | K1 µs | K2/exchange µs | K1 alg. frac | K1 DRAM frac (ncu) | step alg. frac | k'/k | sync GB/s | CPU ref ms |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for (n, n_g, dd, st, k1, k2, fr, dr, sf, dens, nvl, cpu) in rows:
        f = lambda v, fmt: fmt.format(v) if v is not None else "—"
        print(f"| {n} | {n_g / 1e6:g}M | {dd:g} | {st:.1f} | {k1:.1f} | {k2:.1f} | {fr:.2f} | "
              f"{f(dr, '{:.2f}')} | {sf:.2f} | {dens:.2f} | {f(nvl, '{:.0f}')} | {f(cpu, '{:.1f}')} |")


if __name__ == "__main__":
    main()
