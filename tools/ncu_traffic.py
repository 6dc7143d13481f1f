"""profiles/ncu_traffic.json from an ncu launch list (dev tool).

usage: python tools/ncu_traffic.py profiles/r02_bench_launches.csv > profiles/ncu_traffic.json

The launch list is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv` of
`python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-c0 --no-ckpt --no-sweep`;
for each group below the LAST launch sequence of its kernels is summed (per
launch, like bench.py's roofline.achieved)."""
import csv
import json
import sys

GROUPS = {
    "delta_encode": ["delta_encode_ws_kernel"],
    "delta_decode": ["delta_count_kernel", "delta_scan_kernel", "delta_materialize_kernel",
                     "delta_decode_tma_kernel<2, 0>"],
    "cluster_encode": ["fit_sum_kernel", "fit_stats_kernel", "fit_var_fallback_kernel",
                       "fit_var_combine_kernel", "fit_label_kernel",
                       "fit_decide_kernel", "fit_minmax_kernel", "fit_finalize_kernel",
                       "quantize_codes_kernel"],
    "cluster_dequantize": ["dequantize_kernel"],
}


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "")
    return base.split("::")[-1]


def main(path: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = {}
    for r in rows[1:]:
        launches.setdefault(int(r[ii]), {"name": short(r[ki])})[r[mi]] = float(r[vi])
    seq = [launches[i] for i in sorted(launches)]
    out = {"source": f"{path} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum --clock-control none on `python bench.py --steps 2 "
                     "--warmup 3 --no-e2e --no-cpu --no-c0 --no-ckpt --no-sweep`; the last "
                     "timed launch of each)"}
    for g, kernels in GROUPS.items():
        # the last occurrence of the group's first kernel starts its last
        # sequence (block mode: no pre_combine2 between the sum and the stats)
        starts = [i for i, l in enumerate(seq) if l["name"] == kernels[0]
                  and (len(kernels) < 2 or (i + 1 < len(seq) and seq[i + 1]["name"] == kernels[1]))]
        if not starts:
            continue
        i0 = starts[-1]
        picked = [l for l in seq[i0:] if l["name"] in kernels][:len(kernels)]
        rd = sum(l["dram__bytes_read.sum"] for l in picked)
        wr = sum(l["dram__bytes_write.sum"] for l in picked)
        out[g] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "bytes": rd + wr,
                  "kernels": [l["name"] for l in picked]}
        if g == "cluster_encode":
            out[g]["kernel_ns_serialized"] = sum(l["gpu__time_duration.sum"] for l in picked)
            out[g]["note"] = ("x read from HBM 3x (fit sum + sigma interval, labels + window, "
                              "codes) vs 1 algorithmic: traffic/algorithmic = "
                              f"{(rd + wr) / (5.5 * (1 << 30)):.2f}")
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
