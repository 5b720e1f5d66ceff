"""DRAM traffic per kernel class from an ncu launch list with dram__bytes_read/write.

usage: python scripts/traffic_from_ncu.py <launches.csv> <out.json>
Kernel names map to the executor's profiling classes (stn_exec.cpp launch_op); the
output holds, per class, launches, summed DRAM bytes and bytes per launch, which
bench.py reports as roofline.traffic for the dominant class.
"""
import csv
import io
import json
import sys

CLASSES = [  # (substring of the kernel name, class)
    ("k_absorb_direct", "absorb"), ("k_absorb3", "absorb"), ("k_absorb2", "absorb"),
    ("k_absorb_lanes", "absorb"), ("k_gemm_skinny", "gemm_simt"), ("k_sum_ordered", "root"),
    ("stn_chain_", "sweep"), ("k_chain", "sweep"), ("k_sweep", "sweep"), ("k_gemm_tcf", "gemm_tc"),
    ("k_expand_b_raw", "gemm_tc"),
    ("k_absorb_tma", "absorb_tc"), ("k_absorb_tc", "absorb_tc"), ("k_absorb_mma", "absorb_tc"),
    ("k_gemm_tc", "gemm_tc"), ("k_split_a", "gemm_tc"), ("k_expand_b", "gemm_tc"),
    ("k_perm_tiles", "permute"), ("k_gemm_simt", "gemm_simt"), ("k_generic", "generic"),
    ("k_outer", "generic"), ("k_splitk", "generic"), ("k_leaf_gather", "leaf"),
    ("k_root_accumulate", "root"),
]


def main(src, dst):
    text = open(src).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        per.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    out = {}
    for (_, name), m in per.items():
        cls = next((c for s, c in CLASSES if s in name), None)
        if cls is None:
            continue
        o = out.setdefault(cls, {"launches": 0, "dram_bytes": 0.0, "ns": 0.0})
        o["launches"] += 1
        o["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        o["ns"] += m.get("gpu__time_duration.sum", 0)
    for o in out.values():
        o["bytes_per_launch"] = o["dram_bytes"] / o["launches"]
        o["dram_bytes_per_launch"] = o["bytes_per_launch"]
    label = sys.argv[3] if len(sys.argv) > 3 else src
    json.dump({"source": label, "classes": out}, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
