#!/usr/bin/env python
"""DRAM traffic per launch of bench.py's timing classes from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).

  python tools/ncu_traffic.py launches.csv > profiles/ncu_traffic_c3.json

A "launch" of a class is what bench.py's roofline divides by: one V-cycle
(graph replay), one PCG iteration (SpMV+dot and x/r update), one K(x)x
(k_kx_block + k_kx_partials, or the two-pass p1 + gather). The V-cycle count is the number of fine-level post-smoother
launches (k_sellp_red<1, float, 3, ...>, once per V-cycle)."""
import csv
import json
import sys
from collections import defaultdict


def main():
    rows = defaultdict(dict)
    with open(sys.argv[1]) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        d = rows[r["ID"]]
        d["name"] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", "") or 0)
        m = r["Metric Name"]
        if m.startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(
                r["Metric Unit"], 1)
            d["bytes"] = d.get("bytes", 0.0) + v
    cls = defaultdict(float)
    n_vc = n_pcg = n_kx = n_spe_dot = 0
    for d in rows.values():
        n = d["name"]
        b = d.get("bytes", 0.0)
        # fine-level post-smoother: once per V-cycle
        if "k_sellp_red<1, float, 3" in n or "k_sells_red<float, 3" in n or "k_sells_pair<2>" in n:
            n_vc += 1
        if "k_sell_red<1, double, double, 0>" in n or "k_sells64<0" in n:  # PCG q = A p, p.q
            n_pcg += 1
        if "k_kx_p1" in n or "k_kx_p2" in n or "k_kx_block" in n:  # one per K(x)x apply
            n_kx += 1
        if ("k_sell_red<1, double, double, 0>" in n or "k_sells64<0" in n or "k_pcg_update" in n
                or "k_pcg_direction" in n):
            cls["pcg spmv+vectors"] += b
        elif "k_sells64" in n or "k_sell_red<1, double, double, 1>" in n or "k_sell_red<1, double, double, -1>" in n:
            cls["fp64 spmv (start residual, SPE basis)"] += b  # not V-cycle kernels
        elif "k_kx_" in n:
            cls["stiffness K(x)x"] += b
        elif any(k in n for k in ("k_multi_dot", "k_orth_update", "k_lincomb", "k_scale_rsqrt")):
            cls["spe estimator"] += b
        elif any(k in n for k in ("k_sellp", "k_sells", "k_row<", "k_sell<", "k_dense_", "k_diag_scale", "k_to_f64")):
            cls["v-cycle"] += b
    out = {"source": sys.argv[1], "launches": {"v-cycle": n_vc, "pcg spmv+vectors": n_pcg, "stiffness K(x)x": n_kx},
           "dram_bytes_per_launch": {
               "v-cycle": cls["v-cycle"] / max(1, n_vc),
               # bench.py times a PCG iteration as two regions (SpMV+update, direction)
               "pcg spmv+vectors": cls["pcg spmv+vectors"] / max(1, 2 * n_pcg),
               "stiffness K(x)x": cls["stiffness K(x)x"] / max(1, n_kx)},
           "dram_bytes_total": dict(cls)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
