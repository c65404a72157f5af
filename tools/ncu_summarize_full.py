"""Summarise an `ncu --set full` raw CSV (one row per launch) into the metrics the roofline uses.
Usage: python tools/ncu_summarize_full.py raw.csv.gz [title]"""
import csv
import gzip
import sys

src = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else ""
rows = list(csv.reader(gzip.open(src, "rt") if src.endswith(".gz") else open(src)))
hdr, units, data = rows[0], rows[1], rows[2:]
H = {h: i for i, h in enumerate(hdr)}
KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tf32_pipe_%", "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_active_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("smem_tc_%", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("smem_lsu_%", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("l2_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
]
SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def val(r, k):
    if k not in H:
        return float("nan")
    try:
        v = float(r[H[k]].replace(",", ""))
    except ValueError:
        return float("nan")
    return v * SCALE.get(units[H[k]], 1.0)


print(title)
print("%-58s " % "kernel" + " ".join("%14s" % k for k, _ in KEYS))
for r in data:
    name = r[H["Kernel Name"]].replace("pooch::", "").replace("(pooch::GemmParams, CUtensorMap_st, CUtensorMap_st, "
                                                               "CUtensorMap_st, CUtensorMap_st)", "")
    name = name.replace("void ", "").replace("(anonymous namespace)::", "")[:58]
    print("%-58s " % name + " ".join("%14.1f" % val(r, k) for _, k in KEYS))
